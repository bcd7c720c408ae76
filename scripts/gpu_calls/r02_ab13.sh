# a22: 132 KB carveout (L1 124 KB) with a smaller table vs the 164 KB one
set -x
mkdir -p gpurun_out
for v in variants/t1920 variants/t1216 variants/t1152 variants/t1920; do
  KTG_LIB_DIR=$v timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02q_ab.jsonl 2>> gpurun_out/r02q_ab.err
done
