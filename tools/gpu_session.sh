set -x
mkdir -p gpurun_out
for n in 592 148 37; do
for lib in libebcc_gpu.so libebcc_m256.so libebcc_m128.so; do
  EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 300 python tools/machine_ab.py $n >> gpurun_out/r2_mach_ab.log 2>&1
done
done
cat gpurun_out/r2_mach_ab.log | grep fields
export EBCC_GRAPHS=0 EBCC_LANES=1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:machine_kernel" --launch-count 3 \
  -o gpurun_out/r2_machine148 python tools/prof_compress.py 148 1 > gpurun_out/r2_ncu_mach.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:BaseProbeEpi<\(bool\)1>, \(bool\)0, \(bool\)0, \(bool\)1" -s 5 --launch-count 1 \
  -o gpurun_out/r2_l0inc148 python tools/prof_compress.py 148 1 > gpurun_out/r2_ncu_l0.log 2>&1
ls -la gpurun_out
