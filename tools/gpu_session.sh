set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests.log 2>&1
tail -n 3 gpurun_out/r2_gputests.log
EBCC_TRACE=1 timeout 600 python tools/prof_e2e_split.py 2368 > gpurun_out/r2_e2e_trace2.log 2>&1
grep -v "^\[ebcc" gpurun_out/r2_e2e_trace2.log
for L in 2 3; do
EBCC_LANES=$L timeout 900 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/r2_bench_lanes$L.json 2> gpurun_out/r2_bench_lanes$L.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench_lanes$L.json')); print($L, d['value'], d['compress_gbs'], d['decompress_gbs'], d['e2e']['value'], d['e2e']['ms_compress'], d['e2e']['ms_decompress'])"
done
