set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -q -x -k "multi_batch or small_chunk or every_config" > gpurun_out/r2_gputests_dec.log 2>&1
tail -n 2 gpurun_out/r2_gputests_dec.log
for G in 4 8; do
EBCC_DEC_GROUPS=$G timeout 900 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 3 > gpurun_out/r2_bench_g$G.json 2> gpurun_out/r2_bench_g$G.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench_g$G.json')); print($G, d['value'], d['compress_gbs'], d['decompress_gbs'], d['e2e']['value'], d['e2e']['ms_compress'], d['e2e']['ms_decompress'])"
done
