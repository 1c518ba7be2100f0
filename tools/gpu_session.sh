set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ebcot.py -q -x > gpurun_out/r2_ebcot_tests.log 2>&1
tail -n 3 gpurun_out/r2_ebcot_tests.log
timeout 600 python tools/ebcot_bench.py 148 > gpurun_out/r2_ebcot_bench2.log 2>&1
timeout 600 python tools/ebcot_bench.py 37 >> gpurun_out/r2_ebcot_bench2.log 2>&1
grep fields gpurun_out/r2_ebcot_bench2.log
