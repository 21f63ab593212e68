timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_implicit.py tests/test_gpu_fullsize.py -q -x -k "not E_identical and not noisy_configs" 2>&1 | tail -2
XM_VERBOSE=1 timeout 300 python tools/imp_solve.py E 2 2>&1 | grep -E 'cholesky|K\^-1|^build'
XM_PROFILE=0 XM_PHASES=1 timeout 300 python tools/repro_E.py B bsbs 2>&1 | grep -E 'cholesky|certify|^[0-9] s'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_chol_panel --launch-skip 20 --launch-count 3 python tools/imp_solve.py E 1 2>&1 | grep -E 'duration'
