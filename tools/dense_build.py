import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene
sc = config_scene("E")
dev = torch.device("cuda", 0)
ins = [torch.from_numpy(a).to(dev) for a in (sc.frame, sc.landmark, sc.pts, sc.w)]
with xm.Context(implicit_q=0) as ctx:
    for rep in range(3):
        print(f"--- rep {rep}", file=sys.stderr, flush=True)
        torch.cuda.synchronize(); t = time.time(); ctx.build_Q(sc.N, sc.M, *ins); torch.cuda.synchronize()
        print("build", time.time() - t, flush=True)
