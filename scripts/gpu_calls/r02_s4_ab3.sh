# session 4: warp-uniform step loop vs per-lane loop (hit path on (value, rk) payloads, whole-strip variant and hit rings removed) -- parity + A/B; ncu of the load-time fill passes
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py tests/test_gpu_golden_large.py -q -x > gpurun_out/r02x5_parity.log 2>&1
for spec in "--scale 24" "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr"; do
  for v in variants/lanes paper_2009_07929_b200/lib; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02x5_ab.jsonl 2>> gpurun_out/r02x5_ab.err
  done
done
timeout 900 ncu --set full --clock-control none -k regex:"k_fill_all|k_fill_in_all|k_edge_keys" -c 3 -o gpurun_out/r02x5_fill_s24 python scripts/profile_run.py --scale 24 --k 935 > gpurun_out/r02x5_ncu_fill.log 2>&1
