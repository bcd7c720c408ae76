# session 4 final kernels (one-IMAD hash, (value, rk) hit path, warp-uniform step loop, half strips for short batches): full suite, smoke, bench, e2e phases, A/B of 512-element strips, ncu of the pass at s24 / ER, launch list
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02z4_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z4_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02z4_bench.log 2>&1
KTG_LOAD_TIMING=1 timeout 600 python scripts/e2e_phases.py 24 3 935 > gpurun_out/r02z4_e2e_phases.log 2>&1
for spec in "--scale 24" "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr"; do
  for v in paper_2009_07929_b200/lib variants/s512; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02z4_ab.jsonl 2>> gpurun_out/r02z4_ab.err
  done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02z4_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02z4_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02z4_a22_er22 python scripts/profile_run.py --graph er --scale 22 --k 3 --no-degree-bound > gpurun_out/r02z4_ncu_er.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z4_launch_s24.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02z4_launch.log 2>&1
