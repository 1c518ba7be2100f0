set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ebcot.py -q -x > gpurun_out/r2_ebcot_tests.log 2>&1
tail -n 30 gpurun_out/r2_ebcot_tests.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests.log 2>&1
tail -n 3 gpurun_out/r2_gputests.log
