"""World-size-2 gloo worker for tests/test_dist_gloo.py (launched by torchrun).

CPU stand-in for the N > 1 path's host logic: the ncclUniqueId broadcast and
max-over-ranks timing of bench.py, and the band layout of include/xm.h
xm_shard_rows composed with the symmetric stream: each rank holds the lower
trapezoid of its band of rows, forms the row parts of its rows and the column
parts of every row above (a full-length partial), and ONE all-reduce of the
partials must give Q·V; plus the all-reduce of the ‖Q‖² partials (2× the
strictly lower entries + the diagonal), the column-sharded TRSM's
all-gather of packed G = L⁻¹C̄ slices, and the sharded matrix-free product
(landmark / frame shares + a K̄⁻¹ band, five all-reduces).  Exits non-zero on
any mismatch.
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

    # 3. bands tile [0, n); one all-reduce of the band partials reproduces Q·V
    for N, r, kw in ((7, 3, dict(kind="unordered", vis_prob=0.6, sigma_d=0.05)),
                     (70, 1, dict(kind="unordered", vis_prob=0.2)),
                     (137, 5, dict(kind="loop", window=6))):
        sc = make_scene(N, 25 * N, seed=N, **kw)
        dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        n = 3 * N
        f0, f1, nfpr = xm.shard_rows(N, world, rank)
        a, b = 3 * f0, 3 * f1
        V = random_tangent_ambient(N, r, 5)
        band = np.tril(dm.Q)[a:b, :]                     # the lower trapezoid this rank stores
        strict = band.copy()
        strict[np.arange(b - a), np.arange(a, b)] = 0.0  # column parts exclude the diagonal
        part = np.zeros((n, r))
        part[a:b] += band @ V                            # row parts (j ≤ i)
        part += strict.T @ V[a:b]                        # column parts (j < i)
        t = torch.from_numpy(part)
        dist.all_reduce(t)
        ref = dm.Q @ V
        assert np.abs(t.numpy() - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (N, r)
        # ‖Q‖_F² from the trapezoids (assembly's all-reduce, k_sumsq_rows band mode)
        s2 = torch.tensor([2.0 * float(np.sum(strict ** 2)) + float(np.sum(np.diag(dm.Q)[a:b] ** 2))],
                          dtype=torch.float64)
        dist.all_reduce(s2)
        assert abs(float(s2) - dm.normF ** 2) <= 1e-12 * dm.normF ** 2
        # ranks agree on the plan: contiguous, 32-frame aligned, area-balanced
        plan = torch.tensor([f0, f1, nfpr], dtype=torch.int64)
        plans = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(plans, plan)
        spans = [tuple(p.tolist()) for p in plans]
        assert spans[0][0] == 0 and spans[-1][1] == N
        assert all(spans[q][1] == spans[q + 1][0] for q in range(world - 1))
        assert all(s[0] % 32 == 0 for s in spans)
        assert len({s[2] for s in spans}) == 1 and spans[0][2] == max(s[1] - s[0] for s in spans)
        if N >= 128:  # lower-triangle shares within one 32-frame step of equal
            areas = [s[1] ** 2 - s[0] ** 2 for s in spans]
            assert max(areas) - min(areas) <= 2 * 32 * N + 32 * 32
        # 4. column-sharded TRSM (assembly.cu, world > 1): rank p solves columns
        #    [p·w, (p+1)·w) of G = L⁻¹C̄ (w = ⌈n/P⌉ rounded up to 32), packs them
        #    zero-padded to w columns, and ONE all-gather gives every rank all of G
        m = N - 1
        w = -(-(-(-n // world)) // 32) * 32
        c0, c1 = min(n, rank * w), min(n, rank * w + w)
        Cbar = dm.C[1:, :]
        sl = np.zeros((m, w))
        if c1 > c0:
            sl[:, : c1 - c0] = np.linalg.solve(np.tril(dm.L), Cbar[:, c0:c1])
        parts = [torch.zeros(m * w, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(sl.ravel().copy()))
        G = np.zeros((m, n))
        for q in range(world):
            q0, q1 = min(n, q * w), min(n, q * w + w)
            if q1 > q0:
                G[:, q0:q1] = parts[q].numpy().reshape(m, w)[:, : q1 - q0]
        assert np.abs(G - dm.G).max() <= 1e-10 * max(1.0, np.abs(dm.G).max()), ("trsm shard", N)
        # 5. sharded matrix-free product (implicit.cu, world > 1): landmarks and
        #    frames split by measurement count, K̄⁻¹ by an area-balanced 32-row
        #    band of its lower triangle; five all-reduces of zero-padded pass
        #    outputs reproduce Q·V (the passes follow reading C24)
        E = len(sc.frame)
        fr, lmk, w, pts = sc.frame, sc.landmark, sc.w, sc.pts
        order_l = np.lexsort((fr, lmk))
        lm_off = np.searchsorted(lmk[order_l], np.arange(sc.M + 1))
        order_f = np.lexsort((lmk, fr))
        fr_off = np.searchsorted(fr[order_f], np.arange(N + 1))
        split = lambda off, cnt, p: 0 if p <= 0 else (cnt if p >= world else int(np.searchsorted(off[:cnt], E * p // world)))
        k0, k1 = split(lm_off, sc.M, rank), split(lm_off, sc.M, rank + 1)
        f0, f1 = split(fr_off, N, rank), split(fr_off, N, rank + 1)
        mK = N - 1
        bs = lambda p: 0 if p <= 0 else (mK if p >= world else min(mK, max(0, int(round(mK * np.sqrt(p / world) / 32.0)) * 32)))
        ka, kb = bs(rank), max(bs(rank), bs(rank + 1))
        Kinv = np.linalg.inv(dm.K[1:, 1:])
        Vb = V.reshape(N, 3, r)
        z = np.einsum("ea,ear->er", w[:, None] * pts, Vb[fr])              # (wũ)_eᵀ V_i
        Wk = np.bincount(lmk, weights=w, minlength=sc.M)
        inl = (lmk >= k0) & (lmk < k1)
        m = np.zeros((sc.M, r))
        np.add.at(m, lmk[inl], z[inl])
        m[k0:k1] /= Wk[k0:k1, None]
        tm = torch.from_numpy(m); dist.all_reduce(tm); m = tm.numpy()
        inf = (fr >= max(f0, 1)) & (fr < f1)
        b = np.zeros((N, r))
        np.add.at(b, fr[inf], w[inf, None] * (np.einsum("ea,ear->er", pts[inf], Vb[fr[inf]]) - m[lmk[inf]]))
        tb = torch.from_numpy(b); dist.all_reduce(tb); b = tb.numpy()
        L = np.tril(Kinv)[ka:kb]
        strict = L.copy()
        strict[np.arange(kb - ka), np.arange(ka, kb)] = 0.0
        tpart = np.zeros((mK, r))
        tpart[ka:kb] += L @ b[1:]
        tpart += strict.T @ b[1:][ka:kb]
        tt = torch.from_numpy(tpart); dist.all_reduce(tt)
        t = np.zeros((N, r)); t[1:] = -tt.numpy()
        p = np.zeros((sc.M, r))
        np.add.at(p, lmk[inl], w[inl, None] * t[fr[inl]])
        p[k0:k1] = m[k0:k1] + p[k0:k1] / Wk[k0:k1, None]
        tp = torch.from_numpy(p); dist.all_reduce(tp); p = tp.numpy()
        ino = (fr >= f0) & (fr < f1)
        res = w[ino, None] * (np.einsum("ea,ear->er", pts[ino], Vb[fr[ino]]) + t[fr[ino]] - p[lmk[ino]])
        out = np.zeros((N, 3, r))
        np.add.at(out, fr[ino], pts[ino, :, None] * res[:, None, :])
        to = torch.from_numpy(out.reshape(n, r)); dist.all_reduce(to)
        assert np.abs(to.numpy() - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max()), ("implicit shard", N, r)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("GLOO_OK", flush=True)


if __name__ == "__main__":
    main()
