# static row ends for pristine pivots + partial-run flag (fewer dependent loads per pivot); pristine-graph rank split
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02s_tests.log 2>&1
for v in lib variants/prev lib variants/prev; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02s_ab.jsonl 2>> gpurun_out/r02s_ab.err
done
for v in lib variants/prev; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python bench.py --graph er --scale 22 --ks 3,4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02s_er_$(basename $v).log 2>&1
done
KTG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 20 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02s_bench2.log 2>&1
# reference digests on the box's 16 host cores: s20 K=141..199 and the extra s24 K values
cp gpurun_out/golden_box2.json /tmp/golden_box2.json
timeout 1800 python tests/golden/make_golden_large.py --only s20 --kmin 141 --kmax 199 --out /tmp/golden_box2.json > gpurun_out/golden_box2.log 2>&1
cp /tmp/golden_box2.json gpurun_out/golden_box2.json
timeout 5400 python tests/golden/make_golden_large.py --only s24 --out /tmp/golden_box2.json >> gpurun_out/golden_box2.log 2>&1
cp /tmp/golden_box2.json gpurun_out/golden_box2.json
