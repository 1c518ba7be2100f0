for G in 0 1; do echo "== graphs $G"; EBCC_GRAPHS=$G EBCC_PROFILE=1 python tools/prof_compress.py 37 3 2>&1 | grep -E "^compress wall|ebcc profile" | tail -2 | cut -c1-300; done
