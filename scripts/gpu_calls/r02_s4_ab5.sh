# session 4: tail clipping by interleaved 4-ary searches (KTG_A22_LB4) -- parity + A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py tests/test_gpu_golden_large.py tests/test_gpu_corpus.py tests/test_gpu_edge.py -q -x > gpurun_out/r02x7_parity.log 2>&1
for spec in "--scale 24" "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr"; do
  for v in variants/nolb4 paper_2009_07929_b200/lib; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02x7_ab.jsonl 2>> gpurun_out/r02x7_ab.err
  done
done
