# recompute-kernel change: full suite, bench, configs[4] at full size again
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02x_tests.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02x_bench.log 2>&1
timeout 2000 python scripts/cliques.py 26 32 > gpurun_out/r02x_cliques_s26.log 2>&1
echo "cliques rc=$?" >> gpurun_out/r02x_cliques_s26.log
