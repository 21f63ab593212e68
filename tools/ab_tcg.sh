# A/B on one box: full-row persistent tCG vs lower-triangle persistent tCG
# (XM_SYM_TCG) — phase stamps at config B and the bench step at B and E.
for v in "XM_NO_SYM_TCG=1" "XM_SYM_TCG=1"; do
  echo "== $v"
  env $v XM_PHASES=1 timeout 120 python tools/repro_E.py B bs 2>&1 | grep "fused tCG\|^1 s"
  env $v timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', d['value'], d['solve']['hvps'], d['roofline']['launch_ms'])"
  env $v timeout 300 python bench.py --config E --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('E', d['value'], d['solve']['hvps'], d['roofline']['launch_ms'])"
done
