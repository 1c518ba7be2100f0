set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dwt or small_chunk or large or config3" > gpurun_out/r2_gputests_dwt.log 2>&1
tail -n 3 gpurun_out/r2_gputests_dwt.log
for rep in 1 2; do
for lib in libebcc_prev.so libebcc_gpu.so libebcc_ti128.so; do
  EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 300 python tools/machine_ab.py 474 >> gpurun_out/r2_dwt_ab.log 2>&1
done
done
grep fields gpurun_out/r2_dwt_ab.log
export EBCC_GRAPHS=0 EBCC_LANES=1
lib=libebcc_gpu.so
EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 300 python tools/prof_compress.py 148 1 > gpurun_out/r2_plain_dwt.log 2>&1 && \
EBCC_LIB=$PWD/paper_2510_22265_b200/$lib timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_launches_dwt.csv python tools/prof_compress.py 148 1 > gpurun_out/r2_ncu_dwt.log 2>&1
python tools/launch_table.py gpurun_out/r2_launches_dwt.csv 60 | grep lift
