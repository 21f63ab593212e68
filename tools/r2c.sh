XM_VERBOSE=1 python tools/repro_E.py E bb 2>&1 | grep -v "^\s*$" | tail -8
ncu --set full --clock-control none --import-source on -k regex:dgemm_tn --launch-skip 316 --launch-count 1 -o gpurun_out/r2c_syrk_E python tools/repro_E.py E b > gpurun_out/r2c_ncu.log 2>&1
tail -5 gpurun_out/r2c_ncu.log
