set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_large.py -m gpu -q -k "s14_every or s20" > gpurun_out/r02e5_tests.log 2>&1
for v in lib variants/q0 variants/base lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02e5_ab.jsonl 2>> gpurun_out/r02e5_ab.err
done
