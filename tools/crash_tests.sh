echo "== small alone"; timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "small_chunk" 2>&1 | tail -3
echo "== spiht then small"; timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "spiht_prefix or small_chunk" 2>&1 | tail -3
echo "== dwt then small"; timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "dwt_bitwise or small_chunk" 2>&1 | tail -3
