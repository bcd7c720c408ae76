# session 4: next task claimed under the flush barrier (KTG_A22_EARLYCLAIM) -- parity (incl. multi-rank) + A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py tests/test_gpu_group.py tests/test_gpu_peers.py -q -x > gpurun_out/r02x9_parity.log 2>&1
for spec in "--scale 24" "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr"; do
  for v in variants/noearly paper_2009_07929_b200/lib; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02x9_ab.jsonl 2>> gpurun_out/r02x9_ab.err
  done
done
