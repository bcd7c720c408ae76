# new carried-round kernels: full suite, bench, sanitizers
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02h_tests.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02h_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launch_s24_k3.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02h_launch.log 2>&1
bash scripts/gpu_calls/r02_sanitize.sh
