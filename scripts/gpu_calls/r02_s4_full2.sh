# session 4: warp-uniform step loop, match-first probe, precombined working row ends in k_fill_in_all -- full suite, smoke, bench, e2e phases, A/B of the probe order, ncu of the pass + launch list
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02y4_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y4_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02y4_bench.log 2>&1
KTG_LOAD_TIMING=1 timeout 600 python scripts/e2e_phases.py 24 3 935 > gpurun_out/r02y4_e2e_phases.log 2>&1
for v in variants/emptyfirst paper_2009_07929_b200/lib; do
  KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py --scale 24 --tag $v >> gpurun_out/r02y4_ab.jsonl 2>> gpurun_out/r02y4_ab.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_support_a22 -c 1 -o gpurun_out/r02y4_a22_s24 python scripts/profile_run.py --scale 24 --k 3 --no-degree-bound > gpurun_out/r02y4_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02y4_launch_s24.csv python scripts/profile_run.py --scale 24 --k 3 935 > gpurun_out/r02y4_launch.log 2>&1
