# session 4: tail elements per lane per step (KTG_A22_UNROLL 3 / 4 / 5) on the final build -- parity of U=5 + A/B
set -x
mkdir -p gpurun_out
for spec in "--scale 24" "--scale 20 --ks 3,304 --cache /tmp/ktg_s20.ztcsr" "--graph er --scale 22 --ks 3,4 --cache /tmp/ktg_er22.ztcsr"; do
  for v in variants/u3 paper_2009_07929_b200/lib variants/u5; do
    KTG_LIB_DIR=$v timeout 900 python scripts/ab_s24.py $spec --tag $v >> gpurun_out/r02x8_ab.jsonl 2>> gpurun_out/r02x8_ab.err
  done
done
KTG_LIB_DIR=variants/u5 timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_quick.py tests/test_gpu_kat.py -q -x > gpurun_out/r02x8_parity_u5.log 2>&1
