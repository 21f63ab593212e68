"""NEXT-4 throughput: Thm 3's random-initialisation experiment ("1000 trials",
P:474) — B staircases in ONE xm_solve_batch launch vs the single-instance path
(xm_set_factor + xm_solve per trial) on the same GPU.
usage: python tools/batch_bench.py [A|BAL93] [trials]
  A      config A's scene (N = 10: shared-memory layout)
  BAL93  BAL-93-shaped scene (the paper's trials: N = 93, 61203 points, mean
         track 4.7, small noise; global-memory layout)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import xm_oracle as xo
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene, make_scene, random_factor

which = sys.argv[1] if len(sys.argv) > 1 else "A"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
if which == "BAL93":
    sc = make_scene(93, 61203, "unordered", seed=0, track_mean=4.7, sigma_u=1e-3, sigma_d=0.01)
    desc = "BAL-93-shaped (N=93, M=61203, mean track 4.7, sigma_u 1e-3, sigma_d 0.01)"
else:
    sc = config_scene("A")
    desc = "config A (N=10, M=500, noise-free)"
dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
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
X0 = Yg[0][:, :res[0]["r"]] @ Yg[0][:, :res[0]["r"]].T
same = sum(np.linalg.norm(Yg[b][:, :res[b]["r"]] @ Yg[b][:, :res[b]["r"]].T - X0) <= 1e-6 * np.linalg.norm(X0)
           for b in range(B))
print(json.dumps({"scene": desc, "N": sc.N, "E": sc.E, "trials": B,
                  "batched_s": tb, "batched_trials_per_s": B / tb,
                  "single_instance_s_per_trial": ts, "single_trials_per_s": 1 / ts,
                  "speedup": ts * B / tb,
                  "certified": int(sum(r["certified"] for r in res)),
                  "same_X_as_trial_0": int(same),
                  "escalated": int(sum(r["r"] > 3 for r in res)),
                  "mean_hvps": float(np.mean([r["hvps"] for r in res]))}))
