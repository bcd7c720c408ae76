# recompute path (k_support_chunked, the s26 config's kernel): 4 / 5 / 6 CTAs per SM
set -x
mkdir -p gpurun_out
KTG_LIB_DIR=variants/cb6 timeout 900 python -m pytest tests/test_gpu_large.py -q -k "s14_every and recompute or label" > gpurun_out/r02w_parity.log 2>&1
for v in lib variants/cb5 variants/cb6 lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 900 python scripts/ab_s24.py --recompute --tag $v >> gpurun_out/r02w_ab.jsonl 2>> gpurun_out/r02w_ab.err
done
