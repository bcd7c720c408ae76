# session 4: strips 512 / 256 / 128 by batch size (was 256 / 128) -- parity, A/B against the 256-strip build, full suite, bench, ncu of the pass, launch list
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py tests/test_gpu_golden_large.py -q -x > gpurun_out/r02z5_parity.log 2>&1
for spec in "--scale 24" "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr"; do
  for v in variants/adapt1 paper_2009_07929_b200/lib; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02z5_ab.jsonl 2>> gpurun_out/r02z5_ab.err
  done
done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02z5_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z5_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02z5_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02z5_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02z5_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z5_launch_s24.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02z5_launch.log 2>&1
