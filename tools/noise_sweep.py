"""NEXT-4's second workload at the paper's size: App. G's depth-noise sweep
(every observation's depth scaled by (1+ε)^x, x ~ U(−1, 1)) on a
BAL-93-shaped view graph — one Q per noise level, identity starts, ALL levels
(× seeds) in ONE xm_solve_batch launch.  Reports per level: certified, final
rank (3 = the relaxation is tight at the rank-3 optimum), λ_min, f.
usage: python tools/noise_sweep.py [seeds_per_level]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import xm_oracle as xo
from paper_2502_04640_b200 import xm
from synth.scenes import make_scene

levels = [0.0, 0.1, 0.25, 0.5, 1.0, 1.5, 2.0, 3.0, 5.0]
seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Qs, meta = [], []
t0 = time.perf_counter()
for eps in levels:
    for sd in range(seeds):
        sc = make_scene(93, 61203, "unordered", seed=100 + sd, track_mean=4.7, eps=eps)
        Qs.append(xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w).Q)
        meta.append((eps, sd))
t_build = time.perf_counter() - t0
Q = np.stack(Qs)
Y0 = np.zeros((len(Qs), 279, 3))
for i in range(93):
    Y0[:, 3 * i:3 * i + 3, :] = np.eye(3)
with xm.Context() as ctx:
    ctx.solve_batch(Q[:2], Y0[:2])                  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    Yg, res = ctx.solve_batch(Q, Y0)
    torch.cuda.synchronize()
    tb = time.perf_counter() - t
out = {"scene": "BAL-93-shaped (N=93, M=61203, mean track 4.7), App. G depth noise (1+eps)^x",
       "instances": len(Qs), "batched_s": tb, "host_Q_build_s (oracle, not timed in batched_s)": t_build,
       "levels": []}
for eps in levels:
    rs = [res[k] for k, (e, _) in enumerate(meta) if e == eps]
    out["levels"].append({"eps": eps, "certified": int(sum(r["certified"] for r in rs)), "n": len(rs),
                          "rank3": int(sum(r["r"] == 3 for r in rs)),
                          "max_rank": int(max(r["r"] for r in rs)),
                          "lambda_min_rel_min": float(min(r["lambda_min"] / max(1.0, r["normQ"]) for r in rs)),
                          "f_mean": float(np.mean([r["f"] for r in rs])),
                          "mean_hvps": float(np.mean([r["hvps"] for r in rs]))})
print(json.dumps(out))
