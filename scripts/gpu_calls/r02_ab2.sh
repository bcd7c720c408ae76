# group-exchange tests + A/B of the a22 grouping at s24
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_group.py -x -q > gpurun_out/r02b_group.log 2>&1
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_kat.py tests/test_gpu_peers.py tests/test_gpu_quick.py -m gpu -q > gpurun_out/r02b_tests.log 2>&1
for v in lib variants/base variants/g8m4 variants/g1m6 lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02b_ab.jsonl 2>> gpurun_out/r02b_ab.err
done
