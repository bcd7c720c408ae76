# session 4 re-entry: shared-window probe build (c60375e) -- full suite, smoke, bench, ncu of the pass, launch list, sanitizers
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02u_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02u_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02u_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02u_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02u_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02u_launch_s24.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02u_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02u_a22_er22 python scripts/profile_run.py --graph er --scale 22 --k 3 --no-degree-bound > gpurun_out/r02u_ncu_er.log 2>&1
rm -f gpurun_out/r02_san_summary.txt
bash scripts/gpu_calls/r02_sanitize.sh
