# session 3: shared-window probe addressing (no S2R), per-task slot clearing, adaptive strips -- parity + A/B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py -q -x > gpurun_out/r02z_parity.log 2>&1
for spec in "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr" "--scale 24"; do
  for v in variants/base variants/asm variants/asmclear paper_2009_07929_b200/lib; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02z_ab.jsonl 2>> gpurun_out/r02z_ab.err
  done
done
