# a22 table 1,920 + aliased smem: full suite, bench, ncu of the pass (traffic), launch list
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02r_tests.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02r_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02r_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02r_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02r_launch_s24.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02r_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02r_a22_er22 python scripts/profile_run.py --graph er --scale 22 --k 3 --no-degree-bound > gpurun_out/r02r_ncu_er.log 2>&1
