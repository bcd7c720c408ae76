# session 4: one-IMAD (value, run end) hash + funnel-shift filter test (KTG_A22_HASH2), warp-uniform one-pivot fast path (KTG_A22_FAST) -- parity + A/B; e2e phase marks inside the working-layout build
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py tests/test_gpu_corpus.py tests/test_gpu_golden_large.py -q -x > gpurun_out/r02v_parity.log 2>&1
for spec in "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr" "--scale 24"; do
  for v in variants/base variants/h2 paper_2009_07929_b200/lib; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02v_ab.jsonl 2>> gpurun_out/r02v_ab.err
  done
done
KTG_LOAD_TIMING=1 timeout 600 python scripts/e2e_phases.py 24 3 935 > gpurun_out/r02v_e2e_phases.log 2>&1
