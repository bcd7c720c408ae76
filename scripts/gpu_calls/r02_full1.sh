# full GPU suite (incl. reference digests at s24/ER), bench at s24, ncu of the a22 pass, reference arm
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02g_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02g_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02g_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02g_ncu_s24.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_launch_s24_k3.csv python scripts/profile_run.py --scale 24 --k 3 > gpurun_out/r02g_launch_k3.log 2>&1
timeout 2400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02g_ref.log 2>&1
