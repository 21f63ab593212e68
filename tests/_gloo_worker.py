"""World-size-2 gloo worker for tests/test_dist_gloo.py (launched by torchrun).

CPU stand-in for the N > 1 path's host logic: the ncclUniqueId broadcast and
max-over-ranks timing of bench.py, and the row sharding + padded all-gather
layout of include/xm.h xm_shard_rows (each rank multiplies its Q rows, the
shards are all-gathered in rank order, the first n rows must be Q·V), plus the
all-reduce of ‖Q‖² partials.  Exits non-zero on any mismatch.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from oracle import xm_oracle as xo  # noqa: E402
from paper_2502_04640_b200 import xm  # noqa: E402
from synth.scenes import make_scene, random_tangent_ambient  # noqa: E402


def main():
    world, rank, _ = bench.dist_env()
    dist.init_process_group("gloo")
    assert dist.get_world_size() == world == 2

    # 1. id broadcast (bench.share_id): every rank gets rank 0's bytes
    uid = bench.share_id(dist, rank, lambda: bytes(range(128)))
    assert uid == bytes(range(128)), "id broadcast"

    # 2. max over ranks (bench.max_over_ranks)
    assert bench.max_over_ranks(dist, 1.5 + rank, "cpu") == 2.5

    # 3. row shards tile [0, n); padded all-gather reproduces Q·V
    for N, r, kw in ((7, 3, dict(kind="unordered", vis_prob=0.6, sigma_d=0.05)),
                     (10, 1, dict(kind="unordered", vis_prob=0.5)),
                     (37, 5, dict(kind="loop", window=6))):
        sc = make_scene(N, 25 * N, seed=N, **kw)
        dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        n = 3 * N
        f0, f1, nfpr = xm.shard_rows(N, world, rank)
        V = random_tangent_ambient(N, r, 5)
        part = np.zeros((3 * nfpr, r))
        part[: 3 * (f1 - f0)] = dm.Q[3 * f0:3 * f1] @ V
        bufs = [torch.zeros(3 * nfpr, r, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(part))
        full = torch.cat(bufs).numpy()
        assert full.shape[0] == world * 3 * nfpr >= n
        ref = dm.Q @ V
        assert np.abs(full[:n] - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max()), (N, r)
        assert np.all(full[n:] == 0.0)
        # ‖Q‖_F² from per-rank partials (assembly's all-reduce)
        s2 = torch.tensor([float(np.sum(dm.Q[3 * f0:3 * f1] ** 2))], dtype=torch.float64)
        dist.all_reduce(s2)
        assert abs(float(s2) - dm.normF ** 2) <= 1e-12 * dm.normF ** 2
        # ranks agree on the plan
        plan = torch.tensor([f0, f1, nfpr], dtype=torch.int64)
        plans = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(plans, plan)
        spans = [tuple(p.tolist()) for p in plans]
        assert spans[0][0] == 0 and spans[-1][1] == N
        assert all(spans[q][1] == spans[q + 1][0] for q in range(world - 1))
        assert len({s[2] for s in spans}) == 1
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("GLOO_OK", flush=True)


if __name__ == "__main__":
    main()
