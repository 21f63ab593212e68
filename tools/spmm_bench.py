"""Time the Q·V product alone (xm_spmm hook, device buffers, CUDA events in the
library) on a config's Q.  Usage: python tools/spmm_bench.py B [r ...]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "B"
rs = [int(x) for x in sys.argv[2:]] or [1, 3, 4]
sc = config_scene(cfg)
with xm.Context(profile=1) as ctx:
    ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    n = 3 * sc.N
    for r in rs:
        V = torch.randn(n, r, dtype=torch.float64, device="cuda")
        out = torch.empty(n, r, dtype=torch.float64, device="cuda")
        for _ in range(5):
            ctx.spmm(V, out=out)
        ctx.reset_stats()
        for _ in range(50):
            ctx.spmm(V, out=out)
        s = ctx.stats()
        ms = s["spmm_ms"] / max(s["spmm_timed"], 1)
        gbs = s["spmm_alg_bytes"] / max(s["spmm_timed"], 1) / (ms / 1e3) / 1e9
        print(json.dumps({"cfg": cfg, "r": r, "us": round(ms * 1e3, 2), "alg_GBps": round(gbs, 1),
                          "sym": os.environ.get("XM_NO_SYM") is None,
                          "extra": os.environ.get("XM_NVCC_EXTRA", "")}))
