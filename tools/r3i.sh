XM_VERBOSE=1 timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -v '^\s*$' | tail -16
