"""NEXT-4 throughput: Thm 3's random-initialisation experiment ("1000 trials",
P:474) on config A's scene — B staircases in ONE xm_solve_batch launch vs the
single-instance path (xm_set_factor + xm_solve per trial) on the same GPU."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import xm_oracle as xo
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene, random_factor

sc = config_scene("A")
dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
Y0 = np.stack([random_factor(sc.N, 3, 1000 + b) for b in range(B)])
with xm.Context() as ctx:
    ctx.solve_batch(dm.Q, Y0[:8], shared_Q=True)             # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    Yg, res = ctx.solve_batch(dm.Q, Y0, shared_Q=True)
    torch.cuda.synchronize()
    tb = time.perf_counter() - t
    ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    k = 20
    t = time.perf_counter()
    for b in range(k):
        ctx.set_factor(Y0[b])
        ctx.solve()
    torch.cuda.synchronize()
    ts = (time.perf_counter() - t) / k
print(json.dumps({"scene": "config A (N=10, M=500, noise-free)", "trials": B,
                  "batched_s": tb, "batched_trials_per_s": B / tb,
                  "single_instance_s_per_trial": ts, "single_trials_per_s": 1 / ts,
                  "speedup": ts * B / tb,
                  "certified": int(sum(r["certified"] for r in res)),
                  "escalated": int(sum(r["r"] > 3 for r in res)),
                  "mean_hvps": float(np.mean([r["hvps"] for r in res]))}))
