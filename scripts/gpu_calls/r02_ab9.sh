# a22 long tails as warp-uniform items (16-byte loads) vs the flattened strips
set -x
mkdir -p gpurun_out
KTG_LIB_DIR=variants/it96 timeout 900 python -m pytest tests/test_gpu_large.py -q -k "s14_every or s20" > gpurun_out/r02m_it96_parity.log 2>&1
for v in lib variants/it96 variants/it48 variants/it192 lib variants/it96; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02m_ab.jsonl 2>> gpurun_out/r02m_ab.err
done
