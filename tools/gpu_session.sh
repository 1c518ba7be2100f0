set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/r2_gputests.log 2>&1
tail -n 15 gpurun_out/r2_gputests.log
for lib in libebcc_prev.so libebcc_gpu.so; do
  EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 300 python tools/machine_ab.py 474 >> gpurun_out/r2_wide_ab.log 2>&1
done
grep fields gpurun_out/r2_wide_ab.log
