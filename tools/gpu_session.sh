set -x
timeout 300 python tools/host_io_probe.py > gpurun_out/r2_hostio.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2_bfull2.json 2> gpurun_out/r2_bfull2.err
tail -n 5 gpurun_out/r2_bfull2.err
