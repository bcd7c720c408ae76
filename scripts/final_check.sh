timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/f_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref.log 2>&1
timeout 600 python bench.py --mode fixpoint --scale 20 --k 3 > gpurun_out/f_fix.log 2>&1
