# A/B of compile-time variants on one box: per-iteration time of the tCG
# kernel (bench.py roofline launch_ms, profiling events, no phase stamps) and
# the step time at config ${CFG:-B}.  usage: VARIANTS="'' '-DFOO'" bash tools/ab_build.sh
eval "set -- $VARIANTS"
for F in "$@"; do
  XM_NVCC_EXTRA="$F" python -m paper_2502_04640_b200.build > /dev/null
  timeout 300 python bench.py --config ${CFG:-B} --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$F]', d['config']['workload'][:8], 'step', round(d['value'],4), 'hvps', d['solve']['hvps'], 'iter_us', round(d['roofline']['launch_ms']*1e3,2))"
done
python -m paper_2502_04640_b200.build > /dev/null
