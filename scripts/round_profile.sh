set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s3_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k k_support_a22 -c 1 -o gpurun_out/s3_a22 python scripts/profile_run.py --k 3 > gpurun_out/s3_ncu_a22.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k k_support_a22 --csv --log-file gpurun_out/s3_traffic.csv python scripts/traffic_run.py > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_sweep.csv python scripts/profile_sweep.py 3 > gpurun_out/s3_sweep.log 2>&1
