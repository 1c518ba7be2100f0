mkdir -p gpurun_out
EBCC_PROFILE=1 timeout 300 python tools/prof_compress.py 1 4 2>&1 | grep -v slow | tail -4 | cut -c1-200
for n in 1 2; do EBCC_PROFILE=1 timeout 300 python tools/machine_ab.py $n 2>&1 | grep "fields" | tail -3 ; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests.log 2>&1
tail -n 3 gpurun_out/r2_gputests.log
