python -m pytest tests/test_gpu_multirank.py -q -x 2>&1 | tail -15
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not noisy_configs" 2>&1 | tail -3
