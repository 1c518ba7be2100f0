mkdir -p gpurun_out
timeout 900 python tools/prof_configs.py > gpurun_out/r2_all_configs.txt 2>&1
timeout 600 python tools/prof_c4.py >> gpurun_out/r2_all_configs.txt 2>&1
cat gpurun_out/r2_all_configs.txt | grep -v "^\[" | tail -20
