timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
XM_VERBOSE=1 timeout 300 python tools/imp_solve.py E 2 2>&1 | grep -E 'cholesky|^build'
for v in "XM_NO_CHOL_LOOKAHEAD=1" ""; do echo "== [$v]"; env $v XM_PROFILE=0 XM_PHASES=1 timeout 300 python tools/repro_E.py B bsbs 2>&1 | grep -E 'cholesky|^[0-9] s'; done
