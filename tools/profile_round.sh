#!/bin/bash
# Round profile capture (run under gpurun from the repo root):
#  1. launch list of one compress + decompress (ncu gpu__time_duration, graphs
#     off so ncu sees every launch) -> gpurun_out/launches.csv
#  2. ncu --set full of the first base-search level-0 probe (every tile
#     computed) -> gpurun_out/level0_full.ncu-rep
set -x
mkdir -p gpurun_out
EBCC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/prof_compress.py 37 1 > gpurun_out/ncu_launch.log 2>&1
EBCC_GRAPHS=0 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:BaseProbeEpi<\(bool\)1>, \(bool\)0, \(bool\)0, \(bool\)1" --launch-count 1 \
  -o gpurun_out/level0_full python tools/prof_compress.py 37 1 > gpurun_out/ncu_full.log 2>&1
#  3. ncu --set full of the decompress base-stream list machine (the top
#     decompress kernel) -> gpurun_out/machine_dec_full.ncu-rep
EBCC_GRAPHS=0 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:machine_kernel<\(bool\)1>" --launch-count 1 \
  -o gpurun_out/machine_dec_full python tools/prof_compress.py 37 1 > gpurun_out/ncu_mach.log 2>&1
