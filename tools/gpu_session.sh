set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "not every_config" > gpurun_out/r2_gputests_ctl.log 2>&1
tail -n 30 gpurun_out/r2_gputests_ctl.log
timeout 300 python tools/prof_configs.py > gpurun_out/r2_configs_ctl.log 2>&1
timeout 600 python bench.py --fields 296 --steps 3 --no-cpu-baseline > gpurun_out/r2_b296_ctl.json 2> gpurun_out/r2_b296_ctl.err
