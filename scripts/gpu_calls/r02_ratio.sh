# carry/recompute cost-model calibration at s24 + multi-rank bench wiring check (2 ranks sharing the one GPU)
set -x
mkdir -p gpurun_out
RATIO_VAR=KTG_DELTA_RATIO0 CACHE=/tmp/ktg_s24.ztcsr SCALE=24 KS=3,10,30,100,300,935 timeout 1200 python scripts/ratio_scan.py 0.01 0.03 0.1 0.3 1 > gpurun_out/r02j_ratio0.log 2>&1
RATIO_VAR=KTG_DELTA_RATIO FIX0=0.03 CACHE=/tmp/ktg_s24.ztcsr SCALE=24 KS=10,30,100,300,935 timeout 1200 python scripts/ratio_scan.py 0.02 0.0625 0.2 0.6 > gpurun_out/r02j_ratio.log 2>&1
KTG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 20 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02j_bench2.log 2>&1
timeout 900 python bench.py --graph er --scale 22 --ks 3,4 --steps 5 --warmup 3 > gpurun_out/r02j_bench_er22.log 2>&1
timeout 1200 python bench.py --scale 20 --ks all --steps 3 --warmup 3 > gpurun_out/r02j_bench_s20_sweep.log 2>&1
# compute-sanitizer over every engine mode (small graphs, parity-checked).
# Host-loop modes for racecheck / synccheck (the tools do not follow kernels
# launched by conditional CUDA-graph nodes: racecheck aborts the process,
# synccheck flags the first barrier of every graph-launched kernel); the
# graph-launched modes are run separately to document that.
set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
HOST=inc,recompute,label,naive
timeout 1500 $CS --tool memcheck --print-limit 50 --error-exitcode 9 python scripts/sanitize.py --mode all --scale 10 --ks 3,5,9 > gpurun_out/r02_san_memcheck.log 2>&1; echo "memcheck all modes rc=$?" >> gpurun_out/r02_san_summary.txt
timeout 1500 $CS --tool initcheck --print-limit 50 --error-exitcode 9 python scripts/sanitize.py --mode all --scale 10 --ks 3,5,9 > gpurun_out/r02_san_initcheck.log 2>&1; echo "initcheck all modes rc=$?" >> gpurun_out/r02_san_summary.txt
timeout 1500 $CS --tool racecheck --racecheck-report all --print-limit 50 --error-exitcode 9 python scripts/sanitize.py --mode $HOST --scale 10 --ks 3,5,9 --no-api > gpurun_out/r02_san_racecheck.log 2>&1; echo "racecheck host-loop modes rc=$?" >> gpurun_out/r02_san_summary.txt
timeout 1500 $CS --tool synccheck --print-limit 50 --error-exitcode 9 python scripts/sanitize.py --mode $HOST --scale 10 --ks 3,5,9 --no-api > gpurun_out/r02_san_synccheck.log 2>&1; echo "synccheck host-loop modes rc=$?" >> gpurun_out/r02_san_summary.txt
timeout 900 $CS --tool synccheck --print-limit 5 --error-exitcode 9 python scripts/sanitize.py --mode recompute_graph --scale 10 --ks 3 --no-api > gpurun_out/r02_san_synccheck_graph.log 2>&1; echo "synccheck recompute graph mode rc=$?" >> gpurun_out/r02_san_summary.txt
timeout 1200 $CS --tool memcheck --print-limit 50 --error-exitcode 9 python -m pytest tests/test_gpu_group.py -q -k "virtual_ranks_device_resident and 2 or recompute" > gpurun_out/r02_san_group_memcheck.log 2>&1; echo "group memcheck rc=$?" >> gpurun_out/r02_san_summary.txt
