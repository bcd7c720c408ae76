# k_mark without block barriers in its scan loop
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_group.py -q -k "s14_every or group" > gpurun_out/r02u_tests.log 2>&1
for v in lib variants/prev lib variants/prev; do
  d=$v; [ "$v" = lib ] && d=paper_2009_07929_b200/lib
  KTG_LIB_DIR=$d timeout 600 python scripts/ab_s24.py --tag $v >> gpurun_out/r02u_ab.jsonl 2>> gpurun_out/r02u_ab.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02u_launch_s24.csv python scripts/profile_run.py --scale 24 --k 935 > gpurun_out/r02u_launch.log 2>&1
