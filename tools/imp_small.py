import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2502_04640_b200 import xm
from oracle import xm_oracle as xo
from synth.scenes import make_scene, random_tangent_ambient
sc = make_scene(seed=3, N=10, M=500, kind="unordered", vis_prob=0.6)
dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
with xm.Context(implicit_q=1) as ctx:
    ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    print("built", flush=True)
    for r in (4, 3, 1, 5, 7, 12):
        V = random_tangent_ambient(sc.N, r, 40 + r)
        out = ctx.spmm(V)
        print(r, np.linalg.norm(out - dm.Q @ V) / (np.linalg.norm(dm.Q) * np.linalg.norm(V)), flush=True)
