# a22 consecutive-elements mapping / 5 CTAs A/B; group reload fix; multi-rank bench wiring (2 ranks share the GPU)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_group.py -q > gpurun_out/r02k_group.log 2>&1
KTG_LIB_DIR=variants/c4 timeout 900 python -m pytest tests/test_gpu_large.py -q -k "s14_every" > gpurun_out/r02k_c4_parity.log 2>&1
for v in lib variants/c4 variants/b5 variants/c4b5 lib variants/c4; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02k_ab.jsonl 2>> gpurun_out/r02k_ab.err
done
KTG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 20 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02k_bench2.log 2>&1
