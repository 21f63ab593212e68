set -x
OUT=gpurun_out/r4b; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_imp_lm_mean|k_imp_fr_out' \
  --launch-skip 8 --launch-count 2 -o $OUT/ncu_vt -f python tools/imp_prof.py E > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
