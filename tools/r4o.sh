timeout 1200 python bench.py > gpurun_out/r4o_bench_E.json 2> gpurun_out/r4o_bench_E.err; tail -1 gpurun_out/r4o_bench_E.err
python -c "
import json; d=json.load(open('gpurun_out/r4o_bench_E.json')); print(d['value'], d['e2e']['value'], d['phases_ms'], d['roofline']['frac'], d['roofline']['traffic'], d['roofline']['kernel'][:80], d['clocks'], d['gpu_launches'])"
