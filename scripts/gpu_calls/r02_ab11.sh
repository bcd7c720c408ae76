# a22 shared-memory footprint vs L1: aliased step-1/2 arrays, smaller hash tables
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -q -k "s14_every" > gpurun_out/r02o_lib_parity.log 2>&1
KTG_LIB_DIR=variants/t1536 timeout 900 python -m pytest tests/test_gpu_large.py -q -k "s14_every" > gpurun_out/r02o_t1536_parity.log 2>&1
for v in lib variants/nu variants/t1792 variants/t1536 variants/t1280 lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02o_ab.jsonl 2>> gpurun_out/r02o_ab.err
done
