set -x
OUT=gpurun_out/r4a; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "implicit or smoke or edge" 2>&1 | tail -3
for v in "XM_IMP_NO_VT=1" "" ; do echo "== [$v]"; env $v timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -E '^build'; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:'k_imp' --launch-skip 12 --launch-count 12 --log-file $OUT/imp_E.csv python tools/imp_prof.py E > $OUT/ncu.log 2>&1
python tools/ncu_summary.py $OUT/imp_E.csv 2>&1 | head -30 || true
grep -E 'k_imp' $OUT/imp_E.csv | head -40
