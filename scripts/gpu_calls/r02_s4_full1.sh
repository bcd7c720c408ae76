# session 4: default build = one-IMAD hash (KTG_A22_HASH2), fast path removed; fill passes 4 entries per thread -- full suite, smoke, bench, e2e phases, ncu of the pass + launch list
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02w_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02w_bench.log 2>&1
KTG_LOAD_TIMING=1 timeout 600 python scripts/e2e_phases.py 24 3 935 > gpurun_out/r02w_e2e_phases.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02w_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02w_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02w_launch_s24.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02w_launch.log 2>&1
