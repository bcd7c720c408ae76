# session 4 final build: configs[2] (ER 2^22) and configs[1] (s20 K sweep) bench lines
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --graph er --scale 22 --ks 3 > gpurun_out/r02s4_bench_er22.log 2>&1
timeout 1500 python bench.py --scale 20 --ks all --steps 3 --warmup 3 > gpurun_out/r02s4_bench_s20_sweep.log 2>&1
