bash tools/r3b.sh
timeout 600 ncu --set full --clock-control none -k regex:'k_imp_lm_mean|k_imp_fr_out' --launch-skip 20 --launch-count 2 -o gpurun_out/r3d_imp_full python tools/imp_prof.py E > /dev/null 2>&1
ls -la gpurun_out/
