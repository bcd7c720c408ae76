# Round-2 first GPU call: suite sanity, s24/ER ncu of k_support_a22, current s24 fixpoint bench.
set -x
mkdir -p gpurun_out
nproc > gpurun_out/r02e_nproc.txt; lscpu >> gpurun_out/r02e_nproc.txt; free -g >> gpurun_out/r02e_nproc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02e_tests.log 2>&1
timeout 600 python bench.py --mode fixpoint --scale 24 --k 935 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_s24_k935.log 2>&1
timeout 600 python bench.py --mode fixpoint --scale 24 --k 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_s24_k3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k k_support_a22 -c 1 -o gpurun_out/r02e_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02e_ncu_s24.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k k_support_a22 -c 1 -o gpurun_out/r02e_a22_er22 python scripts/profile_run.py --graph er --scale 22 --k 3 --no-degree-bound > gpurun_out/r02e_ncu_er22.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launch_s24_k3.csv python scripts/profile_run.py --scale 24 --k 3 > gpurun_out/r02e_launch_s24.log 2>&1
