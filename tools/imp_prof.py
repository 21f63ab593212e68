import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene, random_tangent_ambient
sc = config_scene(sys.argv[1] if len(sys.argv) > 1 else "E")
with xm.Context(implicit_q=1) as ctx:
    ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    V = random_tangent_ambient(sc.N, 3, 1)
    for _ in range(3):
        ctx.spmm(V)
