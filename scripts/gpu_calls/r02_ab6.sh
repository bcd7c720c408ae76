# a22 smem/L1 split: queue vs no queue, table size, unroll (default carveout)
set -x
mkdir -p gpurun_out
for v in lib variants/q0 variants/q0t10 variants/q1u2 variants/base lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02f_ab.jsonl 2>> gpurun_out/r02f_ab.err
done
KTG_A22_CARVEOUT=50 timeout 600 python scripts/ab_s24.py --tag lib-cv50 >> gpurun_out/r02f_ab.jsonl 2>> gpurun_out/r02f_ab.err
KTG_LIB_DIR=variants/q0t10 KTG_A22_CARVEOUT=25 timeout 600 python scripts/ab_s24.py --tag q0t10-cv25 >> gpurun_out/r02f_ab.jsonl 2>> gpurun_out/r02f_ab.err
