for C in 1 2; do echo "== resid cluster $C"; EBCC_RESID_CLUSTER=$C EBCC_PROFILE=1 python tools/prof_compress.py 37 3 2>&1 | grep -E "^compress wall|ebcc profile" | tail -2 | cut -c1-240; done
