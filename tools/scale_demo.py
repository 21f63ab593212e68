"""NEXT-1's purpose ("removes the 9N² memory wall"): a BAL-Final-
shaped scene far past what a dense Q fits in one B200's 180 GB, solved to a
certificate by the matrix-free products.  Noise-free, so the global optimum is
known (F1): f* = 0 and the rounded poses are the ground truth.
usage: python tools/scale_demo.py [N] [track_mean]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_04640_b200 import xm
from synth.scenes import make_scene

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
track = float(sys.argv[2]) if len(sys.argv) > 2 else 148.0
M = int(round(N * 33782 / 10155))          # config E's points per camera
t = time.perf_counter()
sc = make_scene(N, M, "unordered", seed=0, track_mean=track, track_cap=2000)
t_gen = time.perf_counter() - t
n = 3 * N
dense_Q_GB = 8.0 * n * n / 1e9
free0, total = torch.cuda.mem_get_info()
with xm.Context(implicit_q=1) as ctx:
    torch.cuda.synchronize()
    t = time.perf_counter(); ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w); torch.cuda.synchronize()
    tb = time.perf_counter() - t
    free1, _ = torch.cuda.mem_get_info()
    t = time.perf_counter(); st, info = ctx.solve(); torch.cuda.synchronize(); ts = time.perf_counter() - t
    t = time.perf_counter(); cert = ctx.certify(); torch.cuda.synchronize(); tc = time.perf_counter() - t
    g = ctx.round_recover()
print(json.dumps({"N": N, "M": M, "E": int(sc.E), "n": n, "dense_Q_GB_full_storage": dense_Q_GB,
                  "scene_gen_s": t_gen, "build_s": tb, "solve_s": ts, "certify_s": tc,
                  "device_GB_used_after_build": (free0 - free1) / 1e9, "device_GB_total": total / 1e9,
                  "status": st, "certified": info["certified"], "r": info["r"], "hvps": info["hvps"],
                  "spmms": info["spmms"], "f_rel": info["f"] / info["normQ"], "eta": cert["eta"],
                  "max_R_err": float(np.abs(g["R"] - sc.R).max()), "max_s_err": float(np.abs(g["s"] - sc.s).max())}))
