set -x
mkdir -p gpurun_out
for v in lib variants/base variants/l0 lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02d_ab.jsonl 2>> gpurun_out/r02d_ab.err
done
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_kat.py tests/test_gpu_peers.py tests/test_gpu_quick.py tests/test_gpu_group.py -m gpu -q > gpurun_out/r02d_tests.log 2>&1
