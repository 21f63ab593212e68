"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every tCG path, both streaming kernels, the DMMA
assembly, the fixed-point clique scatter, the certificate (Lanczos, Cholesky
+ shift-invert), rounding and XM².  usage: compute-sanitizer --tool T python tools/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2502_04640_b200 import xm
from synth.scenes import make_scene, random_factor

sc = make_scene(37, 900, "loop", seed=2, window=6, sigma_d=0.02, sigma_u=1e-3, weights="uniform")
for path in ("persist_sym", "persist", "fused", "three_kernel"):
    with xm.Context() as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        Y = random_factor(sc.N, 3, 1)
        eta, Heta, nh, stop = ctx.tcg(Y, 1e3, path)
        print(path, nh, stop, flush=True)
for kw in ({}, {"spmm_kernel": 1}, {"spmm_kernel": 2}, {"scale_reg": 1.0}):
    with xm.Context(**kw) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        st, info = ctx.solve()
        cert = ctx.certify()
        sol = ctx.round_recover()
        keep, nd, nr = ctx.xm2(0.1)
        print(kw, st, info["hvps"], cert["method"], nd, nr, flush=True)
# > 148 frames (every persistent CTA busy, ragged tails), Cholesky + shift-invert certificate
sc2 = make_scene(300, 6000, "loop", seed=3, window=8)
with xm.Context() as ctx:
    ctx.build_Q(sc2.N, sc2.M, sc2.frame, sc2.landmark, sc2.pts, sc2.w)
    st, info = ctx.solve()
    cert = ctx.certify()
    print("loop300", st, info["hvps"], cert["method"], cert["lower_rigorous"], flush=True)
print("SANITIZE_RUN_OK")
