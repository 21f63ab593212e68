timeout 900 python -m pytest tests/test_gpu_implicit.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3h_bench.json 2> gpurun_out/r3h_bench.err; tail -3 gpurun_out/r3h_bench.err
python -c "import json; d=json.load(open('gpurun_out/r3h_bench.json')); print(d['value'], d['config']['mode'], d['phases_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['solve']['eta'], d['other_mode']['value'], d['other_mode']['roofline']['frac'], d['clocks'])"
