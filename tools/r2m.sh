python -m pytest tests/test_gpu_scale_reg.py tests/test_gpu_edge_cases.py -q -x 2>&1 | tail -15
python -m pytest tests/test_gpu_parity.py tests/test_gpu_tcg.py -q -x 2>&1 | tail -3
