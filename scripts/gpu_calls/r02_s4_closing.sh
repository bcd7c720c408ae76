# session 4 closing check of the committed tree: full GPU suite, smoke, bench
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02c_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02c_bench.log 2>&1
