set -x
OUT=gpurun_out/r4g; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "implicit or parity or sym" 2>&1 | tail -2
timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -E '^build'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'k_spmm_sym' --launch-skip 4 --launch-count 3 --log-file $OUT/imp_E.csv python tools/imp_prof.py E > $OUT/ncu.log 2>&1
