# session 3 re-entry: restored tree -- full suite, smoke, bench; a22 baselines at s20 / ER 2^22 / s24
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02y_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02y_bench.log 2>&1
for spec in "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr" "--scale 24"; do
  timeout 900 python scripts/ab_s24.py $spec --tag lib >> gpurun_out/r02y_ab.jsonl 2>> gpurun_out/r02y_ab.err
done
