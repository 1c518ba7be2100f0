set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests.log 2>&1
tail -n 3 gpurun_out/r2_gputests.log
timeout 600 python tools/prof_e2e_split.py 2368 > gpurun_out/r2_e2e_split2.log 2>&1
cat gpurun_out/r2_e2e_split2.log
timeout 1200 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/r2_bench_pf3.json 2> gpurun_out/r2_bench_pf3.err
tail -n 2 gpurun_out/r2_bench_pf3.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench_pf3.json')); print(d['value'], d['compress_gbs'], d['decompress_gbs'], d['e2e'], d['probes'], d['roofline'])"
