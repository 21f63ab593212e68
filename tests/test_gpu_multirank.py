"""The world > 1 (row-sharded) path on ONE GPU, through the C ABI.

`world` contexts in one process, one host thread each, joined by the
loopback group (include/xm.h XM_LOOPBACK_MAGIC) in place of NCCL: band
assembly (each rank the lower trapezoid of its area-balanced band of Q rows,
xm_shard_rows), the lower-triangle stream over the band + ONE all-reduce of
the n×r partials per product, the all-reduce of ‖Q‖², replicated per-camera
work and dots, the world > 1 Lanczos and recovery.  Checked against the oracle with the
end-to-end tolerances of test_gpu_parity.py, and across ranks: every rank
holds the same (bitwise) factor, certificate and recovered solution.
"""
import threading

import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import make_scene, random_tangent_ambient

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


def run_ranks(xm, world, token, fn):
    """fn(ctx, rank) on `world` threads sharing one loopback group."""
    gid = xm.loopback_id(token)
    out, err = [None] * world, [None] * world

    def body(q):
        try:
            with xm.Context(rank=q, world=world, nccl_id=gid) as ctx:
                out[q] = fn(ctx, q)
        except BaseException as e:  # noqa: BLE001 — re-raised below
            err[q] = e

    th = [threading.Thread(target=body, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "loopback ranks deadlocked"
    for e in err:
        if e is not None:
            raise e
    return out


SCENES = [
    dict(N=37, M=900, kind="loop", window=6),                                   # ragged bands
    dict(N=130, M=2500, kind="unordered", track_mean=10.0, zipf=0.8, sigma_d=0.05, sigma_u=1e-3),
    dict(N=300, M=6000, kind="loop", window=8),              # > 2 panels per band, 8 ranks busy
]


def tril_rows(Q, a, b):
    """Rows a..b−1 of Q with the (unstored) entries right of the diagonal as NaN."""
    out = Q[a:b].copy()
    for i in range(b - a):
        out[i, a + i + 1:] = np.nan
    return out


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("cfg", SCENES, ids=lambda c: f"{c['kind']}{c['N']}")
def test_sharded_solve_matches_oracle(xm, cfg, world):
    sc = make_scene(seed=3, **cfg)
    dm, st, sol, rep = xo.solve(sc)
    N, n = sc.N, 3 * sc.N
    V = random_tangent_ambient(N, 3, 17)
    V7 = random_tangent_ambient(N, 7, 18)                  # r > 5: column groups of ≤ 5

    def fn(ctx, q):
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        f0, f1, _ = xm.shard_rows(N, world, q)
        Qrows = ctx.Q_rows(3 * f0, 3 * (f1 - f0)) if f1 > f0 else np.zeros((0, n))
        QV = ctx.spmm(V)
        QV7 = ctx.spmm(V7)
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
        return dict(f0=f0, f1=f1, Qrows=Qrows, QV=QV, QV7=QV7, status=status, info=info,
                    cert=cert, g=g, Y=ctx.get_factor())

    res = run_ranks(xm, world, f"solve-{N}-{world}", fn)
    # the bands tile Q's rows; each rank's lower trapezoid matches the oracle
    Qg = np.concatenate([r["Qrows"] for r in res])
    assert Qg.shape == (n, n)
    Qt = tril_rows(dm.Q, 0, n)
    ok = ~np.isnan(Qt)
    assert np.array_equal(np.isnan(Qg), ~ok)
    assert np.linalg.norm(Qg[ok] - Qt[ok]) <= 1e-10 * dm.normF
    for r in res:
        assert np.linalg.norm(r["QV"] - dm.Q @ V) <= 1e-10 * np.linalg.norm(dm.Q @ V)
        assert np.linalg.norm(r["QV7"] - dm.Q @ V7) <= 1e-10 * np.linalg.norm(dm.Q @ V7)
        assert np.array_equal(r["QV"], res[0]["QV"])     # one all-reduce: identical everywhere
    # replicated state is bitwise identical on every rank
    for r in res[1:]:
        assert np.array_equal(r["Y"], res[0]["Y"])
        assert r["info"]["f"] == res[0]["info"]["f"]
        assert r["cert"]["lambda_min"] == res[0]["cert"]["lambda_min"]
        assert np.array_equal(r["g"]["t"], res[0]["g"]["t"])
    r0 = res[0]
    assert r0["status"] == 0 and r0["info"]["certified"] == 1 and st.certified
    assert abs(r0["info"]["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    Xo = st.Y @ st.Y.T
    Yg = r0["Y"]
    assert np.linalg.norm(Yg @ Yg.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
    assert abs(r0["cert"]["rho_hat"] - sol.rho_hat) <= 1e-8 * (1.0 + abs(sol.rho_hat))
    assert r0["cert"]["eta"] <= 1e-6
    np.testing.assert_allclose(r0["g"]["s"], sol.s, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(r0["g"]["R"], sol.R, atol=1e-6)
    np.testing.assert_allclose(r0["g"]["t"], sol.t, atol=1e-6 * max(1.0, np.abs(sol.t).max()))


def test_more_ranks_than_frames(xm):
    """world > N: trailing ranks own no rows (empty shard) and still take part
    in every collective."""
    sc = make_scene(3, 60, "unordered", seed=2, vis_prob=0.8)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    V = random_tangent_ambient(sc.N, 2, 3)

    def fn(ctx, q):
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        return ctx.spmm(V)

    for QV in run_ranks(xm, 4, "tiny-4", fn):
        assert np.linalg.norm(QV - dm.Q @ V) <= 1e-12 * max(1.0, np.linalg.norm(dm.Q @ V))


@pytest.mark.parametrize("world", [2, 3])
def test_xm2_sharded(xm, world):
    """XM² on the sharded path: every rank ranks the same
    replicated solution's residuals and keeps the same measurements as the
    oracle; each rank rebuilds its own rows of Q from them (gathered Q = the
    oracle's Q of the kept set) and the second solve matches the oracle's."""
    from synth.scenes import corrupt
    sc0 = make_scene(12, 400, "unordered", seed=4, vis_prob=0.5, sigma_u=1e-3, sigma_d=0.01)
    sc, bad = corrupt(sc0, 0.04, seed=4)
    first, okeep, ores, second = xo.xm2(sc)
    dm2, st_o, osol2, rep2 = second

    def fn(ctx, q):
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        ctx.solve(r0=3)
        ctx.round_recover()
        res = ctx.edge_residuals()
        keep, nd, nr = ctx.xm2(0.1)
        lo, hi, _ = xm.shard_rows(sc.N, world, q)
        Qrows = ctx.Q_rows(3 * lo, 3 * (hi - lo)) if hi > lo else np.zeros((0, 3 * sc.N))
        st2, info2 = ctx.solve(r0=3)
        sol2 = ctx.round_recover()
        return res, keep, Qrows, info2, sol2, ctx.get_factor()

    out = run_ranks(xm, world, f"xm2-{world}", fn)
    for q in range(world):
        res, keep, Qrows, info2, sol2, Y = out[q]
        assert np.array_equal(keep, okeep)
        assert np.array_equal(res, out[0][0])                    # replicated, bitwise
        assert np.array_equal(sol2["s"], out[0][4]["s"])
        assert info2["certified"] == 1
        assert abs(info2["f"] - st_o.f) <= 1e-8 * (1.0 + abs(st_o.f))
        assert np.max(np.abs(sol2["R"] - osol2.R)) <= 1e-6
    Qg = np.concatenate([o[2] for o in out], axis=0)
    Qt = tril_rows(dm2.Q, 0, 3 * sc.N)
    ok = ~np.isnan(Qt)
    assert np.array_equal(np.isnan(Qg), ~ok)
    assert np.linalg.norm(Qg[ok] - Qt[ok]) <= 1e-10 * dm2.normF


# ---------------------------------------------------------------- matrix-free (NEXT-1)
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg", SCENES[:2], ids=lambda c: f"{c['kind']}{c['N']}")
def test_sharded_implicit_products_and_solve(xm, cfg, world):
    """The matrix-free products on world > 1: each rank runs its landmark /
    frame share of the passes and its band of K̄⁻¹, five all-reduces per
    product — Q·V (r = 1, 3, 4, 7) ≤ 1e-12‖Q‖‖V‖ against the oracle's Q on
    every rank, and the solve → certificate → recovery against the oracle's
    staircase at the shared tolerance scale, identical on every rank."""
    sc = make_scene(seed=3, **cfg)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    iq = xo.ImplicitQ(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    est = xo.hutchinson_normF(iq.apply, dm.n)
    st = xo.staircase(dm, normQ=est)
    Vs = {r: random_tangent_ambient(sc.N, r, 50 + r) for r in (1, 3, 4, 7)}

    def fn(ctx, q):
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        outs = {r: ctx.spmm(V) for r, V in Vs.items()}
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
        return outs, status, info, cert, g, ctx.get_factor()

    gid = xm.loopback_id(f"imp-{cfg['N']}-{world}")
    out, err = [None] * world, [None] * world

    def body(q):
        try:
            with xm.Context(rank=q, world=world, nccl_id=gid, implicit_q=1) as ctx:
                out[q] = fn(ctx, q)
        except BaseException as e:  # noqa: BLE001
            err[q] = e

    th = [threading.Thread(target=body, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "loopback ranks deadlocked"
    for e in err:
        if e is not None:
            raise e
    for q in range(world):
        outs, status, info, cert, g, Yg = out[q]
        for r, V in Vs.items():
            assert np.linalg.norm(outs[r] - dm.Q @ V) <= 1e-12 * dm.normF * np.linalg.norm(V), (q, r)
        assert status == 0 and info["certified"] == 1 and st.certified
        assert abs(info["normQ"] - est) <= 1e-10 * est
        assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
        Xo = st.Y @ st.Y.T
        assert np.linalg.norm(Yg @ Yg.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
        assert np.array_equal(Yg, out[0][5]), q                      # replicated, bitwise
        np.testing.assert_array_equal(g["t"], out[0][4]["t"])
