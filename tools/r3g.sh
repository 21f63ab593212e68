timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_imp_lm_mean|k_imp_lm_p|k_imp_fr_out|k_imp_fr_b' --launch-skip 8 --launch-count 4 -o gpurun_out/r3g_imp_full python tools/imp_prof.py E > gpurun_out/r3g.log 2>&1
ls -la gpurun_out/ | tail -5
