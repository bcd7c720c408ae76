# session 4: a22 hit path on (value, rk) table payloads (no run re-read, light flag in the pivot word, triangles from the flush) and whole-strip steps without range checks -- parity + A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py tests/test_gpu_corpus.py tests/test_gpu_golden_large.py tests/test_gpu_edge.py -q -x > gpurun_out/r02x4_parity.log 2>&1
for spec in "--scale 24" "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr"; do
  for v in variants/nofs variants/hp_nofs paper_2009_07929_b200/lib; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02x4_ab.jsonl 2>> gpurun_out/r02x4_ab.err
  done
done
