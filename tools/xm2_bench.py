"""Time the XM² step (xm_xm2: residuals at the recovered solution, selection,
restoration, rebuild of Q on the device) and the second solve on a config's
scene with a seeded fraction of outlier measurements (synth.scenes.corrupt).
usage: python tools/xm2_bench.py B:0 E:0.04:1.0 …   (config:outlier fraction[:λ of App. D])"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene, corrupt

for arg in sys.argv[1:] or ["B:0"]:
    parts = arg.split(":")
    cfg = parts[0]
    frac = parts[1] if len(parts) > 1 else "0.04"
    lam = parts[2] if len(parts) > 2 else "0"
    sc, bad = corrupt(config_scene(cfg), float(frac), seed=0)
    with xm.Context(scale_reg=float(lam)) as ctx:
        def timed(fn):
            torch.cuda.synchronize(); t = time.perf_counter(); out = fn(); torch.cuda.synchronize()
            return out, time.perf_counter() - t
        _, tb = timed(lambda: ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w))
        (st, info), ts = timed(lambda: ctx.solve(3))
        _, tr = timed(ctx.round_recover)
        (keep, nd, nr), tx = timed(lambda: ctx.xm2(0.1))
        try:
            (st2, info2), ts2 = timed(lambda: ctx.solve(3))
            cert2, tc2 = timed(ctx.certify)
        except xm.XMError as e:  # e.g. collapsed scales (C18) on long noisy trajectories
            print(json.dumps({"cfg": cfg, "outlier_frac": frac, "scale_reg": lam, "xm2_step_s": round(tx, 4),
                              "dropped": nd, "restored": nr, "solve2_error": str(e)}))
            continue
        print(json.dumps({"cfg": cfg, "outlier_frac": frac, "scale_reg": lam, "E": sc.E, "outliers": int(len(bad)), "dropped": nd, "restored": nr,
                          "outliers_dropped": int((~keep[bad]).sum()), "build_s": round(tb, 4),
                          "solve1_s": round(ts, 4), "status1": st, "xm2_step_s": round(tx, 4),
                          "solve2_s": round(ts2, 4), "status2": st2, "certified2": info2["certified"],
                          "eta2": cert2["eta"], "eta2_rigorous": cert2["eta_rigorous"],
                          "s_min2": info2["s_min"], "f1": info["f"], "f2": info2["f"]}), flush=True)
