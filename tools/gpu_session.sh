set -x
timeout 600 python tools/prof_e2e_c5.py > gpurun_out/r2_e2e_pin.log 2>&1
EBCC_HOSTPIN=0 TAG=nopin timeout 600 python tools/prof_e2e_c5.py > gpurun_out/r2_e2e_nopin.log 2>&1
