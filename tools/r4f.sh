set -x
OUT=gpurun_out/r4f; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "implicit or smoke or edge or multirank or parity" 2>&1 | tail -3
timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -E '^build'
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum --clock-control none --csv \
  -k regex:'k_imp|k_spmm_sym' --launch-skip 24 --launch-count 6 --log-file $OUT/imp_E.csv python tools/imp_prof.py E > $OUT/ncu.log 2>&1
