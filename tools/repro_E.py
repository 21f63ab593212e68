"""Bisect helper: run a sequence of API calls on one context.
usage: python tools/repro_E.py CFG SEQ [key=val scene overrides]   SEQ e.g. "bsbs" (b=build_Q, s=solve, c=certify, r=round)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene
cfg = sys.argv[1]
seq = sys.argv[2] if len(sys.argv) > 2 else "bsbs"
ov = {}
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    ov[k] = float(v) if "." in v or "e" in v else int(v)
sc = config_scene(cfg, **ov)
print(cfg, sc.N, sc.M, sc.E, flush=True)
with xm.Context(profile=int(os.environ.get("XM_PROFILE", "1"))) as ctx:
    for k, op in enumerate(seq):
        t = time.time()
        try:
            if op == "b":
                ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w); msg = ""
            elif op == "s":
                st, info = ctx.solve(3); msg = f"st={st} hvps={info['hvps']} r={info['r']} lz={info['lanczos_steps']}"
            elif op == "c":
                cert = ctx.certify(); msg = f"method={cert['method']}"
            elif op == "r":
                ctx.round_recover(); msg = ""
            print(k, op, "ok", round(time.time() - t, 3), msg, flush=True)
        except Exception as e:
            print(k, op, "FAIL", e, flush=True)
            break
