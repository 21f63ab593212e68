import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import xm_oracle as xo
from paper_2502_04640_b200 import xm
from synth.scenes import make_scene, random_factor
sc = make_scene(93, 61203, "unordered", seed=0, track_mean=4.7, sigma_u=1e-3, sigma_d=0.01)
dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
B = 148
Y0 = np.stack([random_factor(sc.N, 3, 1000 + b) for b in range(B)])
with xm.Context() as ctx:
    ctx.solve_batch(dm.Q, Y0, shared_Q=True)
