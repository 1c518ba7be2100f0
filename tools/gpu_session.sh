set -x
timeout 900 python -m pytest tests/test_gpu_r2.py -x -q > gpurun_out/r2_gputests_r2.log 2>&1
tail -n 5 gpurun_out/r2_gputests_r2.log
for lib in libebcc_gpu.so libebcc_m256.so; do
  EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 300 python tools/machine_ab.py 474 >> gpurun_out/r2_mach_ab.log 2>&1
  EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 300 python tools/machine_ab.py 37 >> gpurun_out/r2_mach_ab.log 2>&1
  EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 300 python tools/machine_ab.py 1 >> gpurun_out/r2_mach_ab.log 2>&1
done
