set -x
OUT=gpurun_out/r4d; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "implicit" 2>&1 | tail -3
for v in "XM_IMP_FPW=1" "XM_IMP_FPW=2" ; do echo "== [$v]"; env $v timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -E '^build'; done
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:'k_imp' --launch-skip 20 --launch-count 5 --log-file $OUT/imp_E.csv python tools/imp_prof.py E > $OUT/ncu.log 2>&1
XM_IMP_FPW=1 timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:'k_imp' --launch-skip 20 --launch-count 5 --log-file $OUT/imp_E1.csv python tools/imp_prof.py E > $OUT/ncu1.log 2>&1
