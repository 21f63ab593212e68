python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -15
timeout 600 python tools/batch_bench.py 1000 2>&1 | tail -2
