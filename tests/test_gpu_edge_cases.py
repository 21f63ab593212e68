"""Degenerate and edge cases of the method on the device, through the C ABI,
against the oracle (and the closed forms that pin it):

* N = 1: Q = 0, the staircase stops at Y = I, certified, λ_min = 0;
* N = 2 (Remark 1): the SDP is tight and the recovered
  relative pose is the scaled (Umeyama) registration — GPU == oracle, and the
  oracle is pinned to the closed form (test_oracle_pins.py);
* single-view landmarks (F10): they add exactly nothing to Q — the
  device Q is BITWISE identical with and without them (their per-edge terms
  cancel exactly: W_k = w_e), and both match the oracle;
* duplicate measurements: first kept, counted.
"""
import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import make_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_single_frame_zero_Q_certified(xm):
    sc = make_scene(1, 7, "unordered", seed=0, vis_prob=1.0)
    dm, st, sol, rep = xo.solve(sc)
    with xm.Context() as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        Qg = ctx.Q_rows(0, 3)
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
    assert np.abs(Qg).max() <= 1e-13 and np.abs(dm.Q).max() <= 1e-13
    assert status == 0 and info["certified"] == 1 and st.certified
    assert abs(info["f"]) <= 1e-13 and abs(cert["lambda_min"]) <= 1e-12
    np.testing.assert_allclose(g["R"][0], np.eye(3), atol=0)
    assert g["s"][0] == 1.0
    # landmarks: p_k = ũ_k (frame 0 is the world frame)
    np.testing.assert_allclose(g["p"], sol.p, atol=1e-12)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_two_frames_match_oracle(xm, seed):
    sc = make_scene(2, 40, "unordered", seed=seed, vis_prob=0.9, sigma_d=0.05, sigma_u=0.01,
                    weights="uniform")
    dm, st, sol, rep = xo.solve(sc)
    with xm.Context() as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        Qg = ctx.Q_rows(0, 6)
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
    assert rel(Qg, dm.Q) <= 1e-10
    assert status == 0 and info["certified"] == 1 and st.certified
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    assert cert["eta"] <= 1e-6
    np.testing.assert_allclose(g["s"], sol.s, rtol=1e-8)
    np.testing.assert_allclose(g["R"], sol.R, atol=1e-7)
    np.testing.assert_allclose(g["t"], sol.t, atol=1e-7 * max(1.0, np.abs(sol.t).max()))


def test_singleton_landmarks_add_exactly_nothing(xm):
    base = make_scene(40, 900, "loop", seed=4, window=6, sigma_d=0.02, sigma_u=1e-3)
    rng = np.random.default_rng(9)
    extra = 50                                            # landmarks seen by one frame only
    src = rng.integers(0, len(base.frame), extra)         # reuse existing (ũ, w): same term bound T
    fr = np.concatenate([base.frame, rng.integers(0, base.N, extra)])
    lm = np.concatenate([base.landmark, base.M + np.arange(extra)])
    pts = np.concatenate([base.pts, base.pts[src]])
    w = np.concatenate([base.w, base.w[src]])
    dm = xo.build_Q(base.N, base.M + extra, fr, lm, pts, w)
    dm0 = xo.build_Q(base.N, base.M, base.frame, base.landmark, base.pts, base.w)
    with xm.Context() as ctx:
        ctx.build_Q(base.N, base.M, base.frame, base.landmark, base.pts, base.w)
        Q0 = ctx.Q_rows(0, 3 * base.N)
        ctx.build_Q(base.N, base.M + extra, fr, lm, pts, w)
        Q1 = ctx.Q_rows(0, 3 * base.N)
        status, info = ctx.solve()
        g = ctx.round_recover() if status == 0 else None
    assert np.array_equal(Q0, Q1)                         # bitwise
    assert rel(Q1, dm.Q) <= 1e-10 and rel(dm.Q, dm0.Q) <= 1e-12
    assert status == 0
    # a singleton landmark is placed at its own observation (Eq. (4)): p_k = s_i R_i ũ + t_i
    i = fr[-1]
    x = g["s"][i] * g["R"][i] @ pts[-1] + g["t"][i]
    np.testing.assert_allclose(g["p"][-1], x, atol=1e-9 * max(1.0, np.abs(x).max()))


def test_duplicates_keep_first(xm):
    sc = make_scene(12, 300, "unordered", seed=2, vis_prob=0.5)
    dup = np.arange(0, len(sc.frame), 7)
    fr = np.concatenate([sc.frame, sc.frame[dup]])
    lm = np.concatenate([sc.landmark, sc.landmark[dup]])
    pts = np.concatenate([sc.pts, sc.pts[dup] * 1.5])     # later duplicates differ: must be dropped
    w = np.concatenate([sc.w, sc.w[dup]])
    dm = xo.build_Q(sc.N, sc.M, fr, lm, pts, w)
    dm0 = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    with xm.Context() as ctx:
        ctx.build_Q(sc.N, sc.M, fr, lm, pts, w)
        Qg = ctx.Q_rows(0, 3 * sc.N)
        st = ctx.stats()
    assert st["n_dup"] == len(dup)
    assert rel(Qg, dm.Q) <= 1e-10 and rel(dm.Q, dm0.Q) <= 1e-12


# ---------------------------------------------------------------- matrix-free (NEXT-1)
def _products(ctx, n, rs=(1, 3, 4, 5, 7)):
    rng = np.random.default_rng(17)
    return {r: (V := rng.standard_normal((n, r)), ctx.spmm(V)) for r in rs}


@pytest.mark.parametrize("case", ["N1", "N2", "singleton", "duplicates"])
def test_implicit_edge_cases(xm, case):
    """The same degenerate inputs through the matrix-free products
    (xm_options.implicit_q): every product Q·V ≤ 1e-12·‖Q‖‖V‖ against the
    oracle's dense Q (r up to 7: the lower-triangle K̄⁻¹ stream and the row
    GEMV), and the solve certifies at the oracle's optimum (N = 1: Q = 0,
    Y = I; N = 2: the tight Umeyama case)."""
    if case == "N1":
        sc = make_scene(1, 7, "unordered", seed=0, vis_prob=1.0)
        fr, lm, pts, w, N, M = sc.frame, sc.landmark, sc.pts, sc.w, sc.N, sc.M
    elif case == "N2":
        sc = make_scene(2, 40, "unordered", seed=1, vis_prob=0.9, sigma_d=0.05, sigma_u=0.01,
                        weights="uniform")
        fr, lm, pts, w, N, M = sc.frame, sc.landmark, sc.pts, sc.w, sc.N, sc.M
    elif case == "singleton":
        base = make_scene(40, 900, "loop", seed=4, window=6, sigma_d=0.02, sigma_u=1e-3)
        rng = np.random.default_rng(9)
        extra = 50
        src = rng.integers(0, len(base.frame), extra)
        fr = np.concatenate([base.frame, rng.integers(0, base.N, extra)])
        lm = np.concatenate([base.landmark, base.M + np.arange(extra)])
        pts = np.concatenate([base.pts, base.pts[src]])
        w = np.concatenate([base.w, base.w[src]])
        N, M = base.N, base.M + extra
    else:
        sc = make_scene(12, 300, "unordered", seed=2, vis_prob=0.5)
        dup = np.arange(0, len(sc.frame), 7)
        fr = np.concatenate([sc.frame, sc.frame[dup]])
        lm = np.concatenate([sc.landmark, sc.landmark[dup]])
        pts = np.concatenate([sc.pts, sc.pts[dup] * 1.5])
        w = np.concatenate([sc.w, sc.w[dup]])
        N, M = sc.N, sc.M
    dm = xo.build_Q(N, M, fr, lm, pts, w)
    st = None
    if N > 1:  # the implicit mode's tolerance scale: the shared Hutchinson estimate (C24)
        iq = xo.ImplicitQ(N, M, fr, lm, pts, w)
        st = xo.staircase(dm, normQ=xo.hutchinson_normF(iq.apply, dm.n))
    with xm.Context(implicit_q=1) as ctx:
        ctx.build_Q(N, M, fr, lm, pts, w)
        prods = _products(ctx, 3 * N)
        status, info = ctx.solve()
        cert = ctx.certify()
    # ≤ 1e-12·‖Q‖‖V‖ plus the rounding floor of forming the per-measurement sums
    # at all, 64·u·T·‖V‖ with T = Σ_e w_e‖ũ_e‖² (N = 1: Q = 0 exactly, the sums
    # A_iV_i − Σ_e (wũ)_e p_kᵀ cancel to rounding)
    T = float(np.sum(w * np.sum(pts * pts, axis=1)))
    u = np.finfo(float).eps / 2
    for r, (V, out) in prods.items():
        tol = (1e-12 * dm.normF + 64 * u * T) * np.linalg.norm(V)
        assert np.linalg.norm(out - dm.Q @ V) <= tol, (case, r)
    assert status == 0 and info["certified"] == 1
    if N == 1:
        assert abs(info["f"]) <= 1e-13 and abs(cert["lambda_min"]) <= 1e-12
    else:
        # N = 2 is tight and converges fast: f to 1e-8; the noisy loop / unordered
        # scenes stop at gradient-tolerance points that agree to the certificate's
        # own precision (η ≤ 1e-6)
        ftol = 1e-8 if case == "N2" else 1e-6
        assert abs(info["f"] - st.f) <= ftol * (1.0 + abs(st.f)), (info["f"], st.f)
        if case == "N2":  # tight (Remark 1): the rounded solution is optimal; the noisy
            # loop of the singleton case certifies at rank 4 with a non-tight relaxation
            # (the oracle's own η = 0.42 there), so η is not small
            assert cert["eta"] <= 1e-6
