import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2502_04640_b200 import xm
from synth.scenes import make_scene, random_tangent_ambient
sc = make_scene(seed=3, N=10, M=500, kind="unordered", vis_prob=0.6)
mode = sys.argv[1]
rng = np.random.default_rng(0)
with xm.Context(implicit_q=1) as ctx:
    ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    r = 4
    V = {"ones": np.ones((30, 4)), "c07": np.full((30, 4), 0.778877), "gauss": rng.standard_normal((30, 4)),
         "int": rng.integers(-3, 3, (30, 4)).astype(float), "rand": random_tangent_ambient(sc.N, r, 44),
         "r5": random_tangent_ambient(sc.N, 5, 44), "r1": random_tangent_ambient(sc.N, 1, 44),
         "r2": random_tangent_ambient(sc.N, 2, 44)}[mode]
    try:
        out = ctx.spmm(V); print(mode, "ok", float(np.abs(out).sum()), flush=True)
    except Exception as e:
        print(mode, "FAIL", e, flush=True)
