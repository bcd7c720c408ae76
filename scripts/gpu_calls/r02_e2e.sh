# where the host-buffer path's time goes at s24
set -x
mkdir -p gpurun_out
KTG_LOAD_TIMING=1 timeout 900 python scripts/e2e_phases.py 24 3 935 > gpurun_out/r02v_e2e_phases.log 2>&1
