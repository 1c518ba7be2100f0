set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests.log 2>&1
tail -n 2 gpurun_out/r2_gputests.log
for n in 474 37 1; do timeout 300 python tools/machine_ab.py $n >> gpurun_out/r2_c15_check.log 2>&1; done
grep fields gpurun_out/r2_c15_check.log
