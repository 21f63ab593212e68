import sys, time, json
sys.path.insert(0, '.')
import numpy as np
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene
for cfg in sys.argv[1:]:
    sc = config_scene(cfg)
    t0 = time.time()
    with xm.Context(profile=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        t1 = time.time()
        st, info = ctx.solve(3)
        t2 = time.time()
        cert = ctx.certify()
        t3 = time.time()
        sol = ctx.round_recover()
        t4 = time.time()
        s = ctx.stats()
    print(cfg, f"build {t1-t0:.3f} solve {t2-t1:.3f} cert {t3-t2:.3f} round {t4-t3:.3f}", "status", st)
    print(json.dumps(info))
    print(json.dumps({k: cert[k] for k in ("lambda_min","rho_hat","rho_dual","eta","lanczos_steps","certified","normQ")}))
    per = s["spmm_ms"]/max(1,s["spmm_timed"]); gbs = s["spmm_alg_bytes"]/max(1,s["spmm_timed"])/(per/1e3)/1e9
    print("spmm per launch ms", per, "GB/s", gbs, "launches", s["kernel_launches"], "spmm_calls", s["spmm_calls"])
    if sc.noise_free: print("max |s-s_gt|", np.abs(sol["s"]-sc.s).max(), "max|R-Rgt|", np.abs(sol["R"]-sc.R).max())
