python -m pytest tests/test_gpu_implicit.py -q -x 2>&1 | tail -20
for v in "" ; do XM_VERBOSE=1 python - <<'PY' 2>&1 | tail -12
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene, random_tangent_ambient
sc = config_scene("E")
with xm.Context(implicit_q=1, profile=1) as ctx:
    t = time.time(); ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w); print("build", time.time() - t, flush=True)
    V = random_tangent_ambient(sc.N, 3, 1)
    ctx.spmm(V); ctx.reset_stats()
    for _ in range(10): ctx.spmm(V)
    st = ctx.stats(); print("spmm calls", st["spmm_calls"], flush=True)
    t = time.time(); s, info = ctx.solve(); print("solve", time.time() - t, s, info["hvps"], info["r"], flush=True)
    t = time.time(); cert = ctx.certify(); print("certify", time.time() - t, cert["eta"], flush=True)
PY
done
