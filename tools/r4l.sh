for v in 0 1 2; do echo "== var $v"; XM_FR_OUT_VAR=$v timeout 300 python tools/imp_solve.py E 2 2>&1 | grep -E '^build' | tail -1
XM_FR_OUT_VAR=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'k_imp_fr_out' --launch-skip 4 --launch-count 2 python tools/imp_prof.py E 2>/dev/null | grep -o 'fr_out<3, [0-9], [0-9]>\|"ns","[0-9,.]*"' | tr '\n' ' '; echo; done
