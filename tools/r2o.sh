python -m pytest tests/test_gpu_xm2.py tests/test_gpu_scale_reg.py tests/test_gpu_edge_cases.py -q -x 2>&1 | tail -4
timeout 1500 python tools/xm2_bench.py E:0 E:0:10 B:0.01:1000 B:0.01:10000 2>&1 | tail -8
