set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -k "rank_partials or support_pass_is_whole or s14_every" > gpurun_out/r02c_tests.log 2>&1
for v in lib variants/base variants/g1 variants/m4 variants/g4 variants/g16 lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02c_ab.jsonl 2>> gpurun_out/r02c_ab.err
done
