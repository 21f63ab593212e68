"""GPU parity for XM² (
reading C22), through the C ABI (xm_edge_residuals, xm_xm2) against the
oracle (oracle.xm_oracle.edge_residuals / xm2_select / xm2)."""
import math

import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import corrupt, make_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


def x_rel_err(Yg, Yo):
    Xg, Xo = Yg @ Yg.T, Yo @ Yo.T
    return np.linalg.norm(Xg - Xo) / np.linalg.norm(Xo)


def _gpu_first(xm, sc):
    ctx = xm.Context(device=0)
    ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    st, info = ctx.solve(r0=3)
    sol = ctx.round_recover()
    return ctx, st, info, sol


def test_edge_residuals_parity(xm):
    """Device residuals vs the oracle's residuals at the oracle's own solution
    (both sides solve the same seeded scene; the solutions agree to ~1e-9, so
    a residual agrees to ~1e-6 of the residual scale); duplicates are NaN;
    the residuals sum to ρ̂ = f(Y₃) of the device's own rounding (F13: Eq. (3)
    at the recovered solution equals trace(Q Ūᵀ Ū))."""
    sc = make_scene(14, 500, "unordered", seed=8, vis_prob=0.5, sigma_u=1e-3, sigma_d=0.02,
                    weights="uniform")
    dm, st, osol, rep = xo.solve(sc)
    ref = xo.edge_residuals(sc.frame, sc.landmark, sc.pts, sc.w, osol)
    # one duplicate measurement appended: ignored by the build, NaN residual
    fr = np.concatenate([sc.frame, sc.frame[:1]])
    lm = np.concatenate([sc.landmark, sc.landmark[:1]])
    pts = np.concatenate([sc.pts, sc.pts[:1] * 1.1])
    w = np.concatenate([sc.w, sc.w[:1]])
    with xm.Context(device=0) as ctx:
        ctx.build_Q(sc.N, sc.M, fr, lm, pts, w)
        st_g, info = ctx.solve(r0=3)
        cert = ctx.certify()
        ctx.round_recover()
        res = ctx.edge_residuals()
    assert st_g == 0 and res.shape == (sc.E + 1,)
    assert np.isnan(res[-1]) and np.all(np.isfinite(res[:-1]))
    assert np.max(np.abs(res[:-1] - ref)) <= 1e-6 * (np.mean(ref) + 1e-300)
    assert abs(res[:-1].sum() - cert["rho_hat"]) <= 1e-9 * (1 + abs(cert["rho_hat"]))
    assert abs(res[:-1].sum() - osol.edge_objective) <= 1e-6 * (1 + osol.edge_objective)


@pytest.mark.parametrize("case", ["outliers", "medium", "restoration"])
def test_xm2_parity(xm, case):
    """Same measurements dropped as the oracle: the masks agree except inside
    groups of equal residuals (e.g. the two measurements of a two-view
    landmark have exactly equal residuals, so the two sides' last-bit
    differences may order them either way); the oracle's residuals of the
    dropped sets then agree value by value.  The second solve agrees with the
    oracle's solve of the same kept set: f ≤ 1e-8(1+|f|), X = YYᵀ ≤ 1e-6
    relative, rotations / scales ≤ 1e-6."""
    if case == "outliers":
        sc0 = make_scene(12, 400, "unordered", seed=4, vis_prob=0.5, sigma_u=1e-3, sigma_d=0.01)
        sc, bad = corrupt(sc0, 0.04, seed=4)
        frac = 0.1
    elif case == "medium":  # > 148 frames: every kernel spans all CTAs, ragged tails
        sc0 = make_scene(150, 3000, "unordered", seed=11, track_mean=8.0, sigma_u=1e-3, sigma_d=0.01)
        sc, bad = corrupt(sc0, 0.03, seed=11)
        frac = 0.1
    else:  # sparse road scene where dropping half the measurements splits the graph;
        # random weights: the two residuals of a two-view landmark differ (no ties)
        sc = make_scene(12, 60, "road", seed=3, sigma_u=1e-3, sigma_d=0.01, track_mean=3.0,
                        weights="uniform")
        frac = 0.5
    if case == "restoration":   # selection + rebuild only (half the measurements dropped)
        dm1, st1, osol, _ = xo.solve(sc)
        ores = xo.edge_residuals(sc.frame, sc.landmark, sc.pts, sc.w, osol)
        okeep = xo.xm2_select(sc.N, sc.M, sc.frame, sc.landmark, ores, frac)
        k = okeep
        second = (xo.build_Q(sc.N, sc.M, sc.frame[k], sc.landmark[k], sc.pts[k], sc.w[k]),)
    else:
        first, okeep, ores, second = xo.xm2(sc, drop_fraction=frac)
    ctx, st, info, sol = _gpu_first(xm, sc)
    with ctx:
        assert st == 0
        keep, n_drop, n_rest = ctx.xm2(frac)
        nd = math.floor(frac * sc.E)
        assert n_drop + n_rest == nd and (~keep).sum() == n_drop
        assert n_rest == nd - (~okeep).sum()         # as many restored as the oracle
        assert (n_rest > 0) == (case != "outliers")
        assert (~keep).sum() == (~okeep).sum()
        a, b = np.sort(ores[~keep]), np.sort(ores[~okeep])
        assert np.all(np.abs(a - b) <= 1e-9 * np.maximum(np.abs(b), 1e-12)), (a, b)
        assert np.array_equal(keep, okeep)           # no ties near the cut in these scenes
        if case != "restoration":
            assert keep[bad].mean() < 0.2            # the outliers are among the dropped
        assert xo.connected_components(sc.N, sc.M, sc.frame[keep], sc.landmark[keep]) == 1
        # reading C22b: every frame keeps ≥ 3 measurements of landmarks seen ≥ 2
        # times, or (best effort) all of its measurements
        kc = np.bincount(sc.landmark[keep], minlength=sc.M)
        for i in range(sc.N):
            mine = sc.frame == i
            assert np.sum(keep & mine & (kc[sc.landmark] >= 2)) >= 3 or keep[mine].all() or \
                np.all(keep[mine] | (kc[sc.landmark[mine]] == 0)), i
        # the rebuilt Q is the data matrix of the kept measurements (= the oracle's second Q)
        Qg = ctx.Q_rows(0, 3 * sc.N)
        dmk = second[0]
        assert np.linalg.norm(Qg - dmk.Q) <= 1e-10 * dmk.normF
        if case == "restoration":
            return
        st2, info2 = ctx.solve(r0=3)
        cert2 = ctx.certify()
        sol2 = ctx.round_recover()
        Yg = ctx.get_factor()
        res2 = ctx.edge_residuals()
    dm2, st_o, osol2, rep2 = second                 # same kept set (asserted above)
    assert st2 == 0 and info2["certified"] == 1 and st_o.certified
    assert abs(info2["f"] - st_o.f) <= 1e-8 * (1.0 + abs(st_o.f))
    assert x_rel_err(Yg, st_o.Y) <= 1e-6
    assert np.max(np.abs(sol2["s"] - osol2.s)) <= 1e-6
    assert np.max(np.abs(sol2["R"] - osol2.R)) <= 1e-6
    assert np.all(np.isnan(res2[~keep])) and np.all(np.isfinite(res2[keep]))
    assert cert2["eta"] <= 1e-6


def test_xm2_matrix_free_rebuild_matches_dense(xm):
    """XM² through the matrix-free products (the E headline mode): the rebuild
    changes E / M at the same device addresses, so every captured tCG graph
    must be recaptured (graph signature) — regression for stale graphs; the
    second solve then equals the dense path's (same kept set, same certified
    optimum) and the oracle's second solve of that kept set."""
    sc0 = make_scene(150, 3000, "unordered", seed=11, track_mean=8.0, sigma_u=1e-3, sigma_d=0.01)
    sc, bad = corrupt(sc0, 0.03, seed=11)
    out = {}
    for imp in (0, 1):
        with xm.Context(device=0, implicit_q=imp) as ctx:
            ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
            st, info = ctx.solve(r0=3)
            ctx.round_recover()
            keep, nd, nr = ctx.xm2(0.1)
            st2, info2 = ctx.solve(r0=3)
            cert2 = ctx.certify()
            out[imp] = (st, keep, st2, info2, cert2, ctx.get_factor())
    (s0, k0, s20, i20, c20, Y0), (s1, k1, s21, i21, c21, Y1) = out[0], out[1]
    assert s0 == s1 == 0 and np.array_equal(k0, k1)
    assert s20 == s21 == 0 and i20["certified"] == i21["certified"] == 1
    assert abs(i21["f"] - i20["f"]) <= 1e-8 * (1.0 + abs(i20["f"]))
    X0, X1 = Y0 @ Y0.T, Y1 @ Y1.T
    assert np.linalg.norm(X1 - X0) <= 1e-6 * np.linalg.norm(X0)
    k = k1
    dm2 = xo.build_Q(sc.N, sc.M, sc.frame[k], sc.landmark[k], sc.pts[k], sc.w[k])
    st_o = xo.staircase(dm2)
    assert abs(i21["f"] - st_o.f) <= 1e-8 * (1.0 + abs(st_o.f))
