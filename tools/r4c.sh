set -x
OUT=gpurun_out/r4c; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "implicit or smoke or edge or multirank" 2>&1 | tail -3
for v in "" ; do echo "== [$v]"; env $v timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -E '^build'; done
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum --clock-control none --csv \
  -k regex:'k_imp' --launch-skip 12 --launch-count 6 --log-file $OUT/imp_E.csv python tools/imp_prof.py E > $OUT/ncu.log 2>&1
grep -E 'k_imp' $OUT/imp_E.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-40,200-
