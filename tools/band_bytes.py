"""Per-rank Q bytes and time per product of the world > 1 band layout at a
BASELINE config, measured with the loopback group on ONE GPU (the ranks'
cooperative band kernels serialise on the device, so each rank's CUDA-event
time is its kernel alone; the loopback all-reduce goes through the host and
is excluded).  usage: python tools/band_bytes.py E 2 4 8"""
import json, os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene, random_tangent_ambient

cfg = sys.argv[1] if len(sys.argv) > 1 else "E"
sc = config_scene(cfg)
for world in [int(w) for w in sys.argv[2:]] or [2]:
    gid = xm.loopback_id(f"bytes-{cfg}-{world}")
    out = [None] * world

    def body(q):
        with xm.Context(rank=q, world=world, nccl_id=gid, profile=1) as ctx:
            ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
            V = random_tangent_ambient(sc.N, 3, 1)
            ctx.spmm(V)
            ctx.reset_stats()
            for _ in range(5):
                ctx.spmm(V)
            st = ctx.stats()
            f0, f1, _ = xm.shard_rows(sc.N, world, q)
            out[q] = dict(rank=q, frames=[f0, f1], alg_bytes=st["spmm_alg_bytes"] / max(st["spmm_timed"], 1),
                          ms=st["spmm_ms"] / max(st["spmm_timed"], 1))

    th = [threading.Thread(target=body, args=(q,)) for q in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    n = 3 * sc.N
    print(json.dumps({"config": cfg, "world": world, "one_gpu_lower_triangle_GB": 8 * n * (n + 1) / 2 / 1e9,
                      "ranks": [dict(r, GB=r["alg_bytes"] / 1e9, GBps=r["alg_bytes"] / r["ms"] / 1e6 if r["ms"] else None)
                                for r in out]}), flush=True)
