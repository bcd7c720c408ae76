set -x
mkdir -p gpurun_out
KTG_LIB_DIR=variants/is96 timeout 900 python -m pytest tests/test_gpu_large.py -q -k "s14_every" > gpurun_out/r02n_is96_parity.log 2>&1
for v in lib variants/is96 variants/is256 variants/is32 lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02n_ab.jsonl 2>> gpurun_out/r02n_ab.err
done
