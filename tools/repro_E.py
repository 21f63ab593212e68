"""Repeated build+solve on config E in one context (bench-like), reporting which step fails."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene
cfg = sys.argv[1] if len(sys.argv) > 1 else "E"
dev_inputs = "--host" not in sys.argv
sc = config_scene(cfg)
ins = (sc.frame, sc.landmark, sc.pts, sc.w)
if dev_inputs:
    ins = tuple(torch.from_numpy(a).cuda() for a in ins)
with xm.Context(profile=1) as ctx:
    for k in range(4):
        t = time.time()
        try:
            ctx.build_Q(sc.N, sc.M, *ins)
            st, info = ctx.solve(3)
            cert = ctx.certify()
            print(k, "ok", st, round(time.time() - t, 3), info["hvps"], info["f"], cert["method"], flush=True)
        except Exception as e:
            print(k, "FAIL", e, flush=True)
            break
