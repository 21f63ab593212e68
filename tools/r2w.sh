python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_multirank.py tests/test_gpu_xm2.py -q -x 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -q -x -k "B_end or E_noisy or E_noise_free" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases_ms'], d['solve']['hvps'], d['clocks'])"
