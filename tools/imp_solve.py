import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene
sc = config_scene(sys.argv[1] if len(sys.argv) > 1 else "E")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
with xm.Context(implicit_q=1) as ctx:
    for rep in range(reps):
        print(f"--- rep {rep}", file=sys.stderr, flush=True)
        t = time.time(); ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w); tb = time.time() - t
        t = time.time(); s, info = ctx.solve(); print("build", tb, "solve", time.time() - t, info["hvps"], info["spmms"], flush=True)
