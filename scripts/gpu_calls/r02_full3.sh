# compaction fix: suite, bench, launch list, sanitizers; then configs[4] at full size (s26/ef32 + cliques)
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02i_tests.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02i_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_launch_s24.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02i_launch.log 2>&1
bash scripts/gpu_calls/r02_sanitize.sh
free -g > gpurun_out/r02i_free.txt
timeout 2700 python scripts/cliques.py 26 32 > gpurun_out/r02i_cliques_s26.log 2>&1
echo "cliques rc=$?" >> gpurun_out/r02i_cliques_s26.log
