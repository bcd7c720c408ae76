# reference digests (oracle/_ref, the unmodified reference) for the upper half of the s20 K sweep, on the box's host cores
set -x
cp gpurun_out/golden_s20_hi.json /tmp/golden_s20_hi.json
timeout 5400 python tests/golden/make_golden_large.py --only s20 --kmin 200 --kmax 305 --out /tmp/golden_s20_hi.json > gpurun_out/golden_s20_hi.log 2>&1
cp /tmp/golden_s20_hi.json gpurun_out/golden_s20_hi.json
