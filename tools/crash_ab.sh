echo "== current"; python -X faulthandler tools/repro_small.py 2>&1 | tail -4
echo "== current overlap0"; EBCC_OVERLAP=0 python -X faulthandler tools/repro_small.py 2>&1 | tail -4
echo "== head lib"; EBCC_LIB=variants/lib_head.so python -X faulthandler tools/repro_small.py 2>&1 | tail -4
