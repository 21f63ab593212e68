python -m pytest tests -m gpu -q --durations=15 2>&1 | tail -25
XM_FULL_PARITY=1 timeout 2000 python -m pytest tests/test_gpu_fullsize.py -q -k "noisy_configs or random_init" -v --durations=5 > gpurun_out/r2_full_parity.log 2>&1; tail -12 gpurun_out/r2_full_parity.log
