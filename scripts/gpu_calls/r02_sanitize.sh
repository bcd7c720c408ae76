# compute-sanitizer over every engine mode (small graphs, parity-checked).
set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  api=""; [ $tool = racecheck ] && api="--no-api"   # racecheck aborts on the pinned result pool (host side)
  timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize.py --mode all --scale 10 --ks 3,5,9 $api > gpurun_out/r02_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02_san_summary.txt
done
timeout 1200 $CS --tool memcheck --print-limit 50 --error-exitcode 9 python -m pytest tests/test_gpu_group.py -q -k "virtual_ranks_device_resident and 2 or recompute" > gpurun_out/r02_san_group_memcheck.log 2>&1
echo "group memcheck rc=$?" >> gpurun_out/r02_san_summary.txt
