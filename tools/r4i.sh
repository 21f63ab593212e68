set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or implicit or fullsize or cert or multirank" 2>&1 | tail -2
for v in "XM_NO_TRSM_FORK=1" "" ; do echo "== [$v]"; env $v timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -E '^build'; env $v python tools/dense_build.py 2>&1 | tail -2; done
