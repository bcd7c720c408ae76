# A/B of a22 task grouping + delta S=0 skip at s24; quick parity suite on the new build.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_kat.py tests/test_gpu_peers.py tests/test_gpu_quick.py -m gpu -x -q > gpurun_out/r02a_tests.log 2>&1
for v in lib variants/base variants/g8m4 variants/g1m6 lib; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02a_ab.jsonl 2>> gpurun_out/r02a_ab.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a_launch_s24_k935.csv python scripts/profile_run.py --scale 24 --k 935 > gpurun_out/r02a_launch_k935.log 2>&1
