for L in 1 2 3 4 6; do echo "== lanes $L"; EBCC_LANES=$L python tools/prof_compress.py 37 3 2>&1 | grep "^compress wall" | tail -1 | cut -c1-200; done
