python -m pytest tests/test_gpu_edge_cases.py -q -x 2>&1 | tail -15
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -k "noisy_configs or random_init or identical_Q" --durations=10 2>&1 | tail -30
