# a22: table size at the 164 KB carveout; long-tail items under the carveout step
set -x
mkdir -p gpurun_out
for v in lib variants/t1792 variants/t1856 variants/t1920 variants/u1_96 variants/u2_96 variants/u2_64t1536 variants/t1920; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02p_ab.jsonl 2>> gpurun_out/r02p_ab.err
done
