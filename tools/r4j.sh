set -x
OUT=gpurun_out/r4j; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > $OUT/bench_E.json 2> $OUT/bench_E.err; tail -2 $OUT/bench_E.err
timeout 600 python bench.py --config B --no-cpu-baseline > $OUT/bench_B.json 2> $OUT/bench_B.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref_E.json 2> $OUT/bench_ref_E.err
python - <<'PY'
import json
for f in ['bench_E','bench_B','bench_ref_E']:
    d=json.load(open(f'gpurun_out/r4j/{f}.json')); print(f, d.get('value'), d.get('e2e',{}).get('value'), d.get('phases_ms'), d.get('roofline',{}).get('frac'), d.get('clocks'))
PY
