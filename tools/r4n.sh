OUT=gpurun_out/r4n; mkdir -p $OUT
# one r = 3 product's six kernels (the first 4 products are the r = 4 Hutchinson probes: 4 × 5 k_imp + 4 spmm_sym = 24 launches)
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_imp_vt|k_imp_lm_mean|k_imp_fr_b|k_spmm_sym|k_imp_lm_p|k_imp_fr_out' \
  --launch-skip 24 --launch-count 6 -o $OUT/ncu_full_imp_E -f python tools/imp_prof.py E > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py $OUT/ncu_full_imp_E.ncu-rep
