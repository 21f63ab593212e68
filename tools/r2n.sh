python -m pytest tests/test_gpu_xm2.py tests/test_gpu_scale_reg.py tests/test_gpu_edge_cases.py -q -x 2>&1 | tail -15
timeout 900 python tools/xm2_bench.py E:0 B:0.01 B:0.01:100 E:0.01 2>&1 | tail -8
