# a22 memory-hint A/B: L2 prefetch of tail starts, S reds evict_first, tail loads evict_last, read-only path
set -x
mkdir -p gpurun_out
for v in lib variants/pf variants/rh variants/lh variants/nc lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02l_ab.jsonl 2>> gpurun_out/r02l_ab.err
done
