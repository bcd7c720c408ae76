# session 4: the s24 reference digests with K=10 added (K = 3, 10, 30, 100, 300, 935, 936) against the final build
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_golden_large.py -q -k s24 > gpurun_out/r02s4_golden_s24.log 2>&1
