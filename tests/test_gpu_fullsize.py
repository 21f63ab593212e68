"""Full-size parity: BASELINE.json configs B (the bench workload) and E (the
north_star target), in the launch configuration bench.py times (default
options ⇒ the same (N, r) kernel choice).

* B (N=2000): the dense oracle still fits — S pattern bit-exact, Q ≤ 1e-10,
  single SpMM on an identical Q ≤ 1e-12, and the whole solve → certificate →
  round/recover against the oracle's (tolerances as test_gpu_parity.py).
* E (N=10155, ~5M observations): no dense n×n oracle.  Sampled rows of Q and
  of Q·V against the oracle's row-wise Schur complement (oracle.q_rows), and
  properties that hold at any size: the known global optimum of a noise-free
  scene (F1), a certified zero duality gap (Eq. (13)), Eq. (3) evaluated at the
  recovered (s, R, t, p) equal to ρ̂, and first-order optimality of the
  recovered t, p (Eq. (4)).
"""
import os

import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import config_scene, random_tangent_ambient

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ----------------------------------------------------------------------------- B
@pytest.fixture(scope="module")
def B(xm):
    sc = config_scene("B")
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    return sc, dm


def test_B_pattern_and_Q(xm, B):
    sc, dm = B
    with xm.Context(profile=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        rowptr, colidx = ctx.S_pattern()
        ro, co = xo.s_pattern(sc.N, dm.frame, dm.landmark)
        np.testing.assert_array_equal(rowptr, ro)
        np.testing.assert_array_equal(colidx, co)
        Qg = ctx.Q_rows(0, 3 * sc.N)
        assert np.array_equal(Qg, Qg.T)
        assert rel(Qg, dm.Q) <= 1e-10
        # Q·V on the GPU-built Q, r = 1 (Lanczos) and r = 3 (tCG)
        for r in (1, 3):
            V = random_tangent_ambient(sc.N, r, 7 + r)
            assert rel(ctx.spmm(V), dm.Q @ V) <= 1e-10


@pytest.mark.parametrize("kernel", [0, 1, 2], ids=["auto", "fullrow", "lowertri"])
def test_B_spmm_identical_Q(xm, B, kernel):
    sc, dm = B
    with xm.Context(profile=1, spmm_kernel=kernel) as ctx:
        ctx.set_Q(dm.Q)
        for r in (1, 3, 4):
            V = random_tangent_ambient(sc.N, r, 11 + r)
            out = ctx.spmm(V)
            ref = dm.Q @ V
            assert rel(out, ref) <= 1e-12, (r, rel(out, ref))


def test_B_end_to_end_vs_oracle(xm, B):
    sc, dm = B
    st = xo.staircase(dm)
    sol = xo.round_recover(dm, st.Y)
    with xm.Context(profile=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        status, info = ctx.solve()
        cert = ctx.certify()
        gsol = ctx.round_recover()
        Yg = ctx.get_factor()
    assert status == 0 and info["certified"] == 1 and st.certified
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    Xo = st.Y @ st.Y.T
    assert np.linalg.norm(Yg @ Yg.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
    assert abs(cert["rho_hat"] - sol.rho_hat) <= 1e-8 * (1.0 + abs(sol.rho_hat))
    assert cert["eta"] <= 1e-6
    np.testing.assert_allclose(gsol["s"], sol.s, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(gsol["R"], sol.R, atol=1e-6)
    np.testing.assert_allclose(gsol["t"], sol.t, atol=1e-6 * max(1.0, np.abs(sol.t).max()))
    assert gsol["n_flipped"] == sol.n_flipped


# ----------------------------------------------------------------------------- E
def _sample_rows(N, k, seed):
    """Rows of the first / last frame, frames at both shard and tile edges,
    and random frames (all three rows of each)."""
    rng = np.random.default_rng(seed)
    frames = np.unique(np.concatenate([[0, 1, N // 2, N - 2, N - 1], rng.integers(0, N, k)]))
    return np.sort((3 * frames[:, None] + np.arange(3)).ravel())


@pytest.fixture(scope="module")
def E_noisy():
    """Config E's shape with keypoint/depth noise (C's noise levels)."""
    return config_scene("E", sigma_u=1e-3, sigma_d=0.01)


def test_E_sampled_Q_rows_and_spmm(xm, E_noisy):
    sc = E_noisy
    rows = _sample_rows(sc.N, 12, 3)
    info = {}
    QI = xo.q_rows(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w, rows, info=info)
    # reading C13: both sides solve with K̄ by backward-stable Cholesky, so
    # ‖ΔQ_I‖ ≲ c·u·κ(K̄)·‖S_I‖ (Q_I is S_I minus a term of S_I's size); c = 8
    # covers both sides' errors.  Config E: κ₁(K̄) ≈ 2.3e4, ‖S_I‖/‖Q_I‖ ≈ 71.
    tol = max(1e-10, 8 * np.finfo(float).eps * info["kappa_K"] * info["S_I_norm"]
              / np.linalg.norm(QI))
    Vs = {r: random_tangent_ambient(sc.N, r, 21 + r) for r in (1, 3)}
    outs = {}
    for kernel in (0, 1, 2):
        with xm.Context(profile=1, spmm_kernel=kernel, implicit_q=0) as ctx:
            ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
            if kernel == 0:
                Qg = np.concatenate([ctx.Q_rows(int(a), 3) for a in rows[::3]])
                assert rel(Qg, QI) <= tol, (rel(Qg, QI), tol)
            for r, V in Vs.items():
                outs[kernel, r] = ctx.spmm(V)
    for r, V in Vs.items():
        ref = QI @ V
        for kernel in (0, 1, 2):
            assert rel(outs[kernel, r][rows], ref) <= tol, (kernel, r, tol)
        # the two streaming kernels on the same GPU-built Q: fp64 rounding apart
        assert rel(outs[1, r], outs[2, r]) <= 1e-12


def test_E_noise_free_known_optimum(xm):
    """F1: noise-free ⇒ f* = 0, certified, rounded poses = ground truth."""
    sc = config_scene("E")
    assert sc.noise_free
    with xm.Context(profile=1, implicit_q=0) as ctx:  # the dense path (matrix-free: test_gpu_implicit)
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        status, info = ctx.solve()
        cert = ctx.certify()
        gsol = ctx.round_recover()
    assert status == 0 and info["certified"] == 1
    assert abs(info["f"]) <= 1e-8 * info["normQ"]
    assert cert["eta"] <= 1e-6
    np.testing.assert_allclose(gsol["s"], sc.s, atol=1e-7)
    np.testing.assert_allclose(gsol["R"], sc.R, atol=1e-7)
    np.testing.assert_allclose(gsol["t"], sc.t, atol=1e-6 * max(1.0, np.abs(sc.t).max()))


def test_E_noisy_certified_and_recovery_optimal(xm, E_noisy):
    sc = E_noisy
    with xm.Context(profile=1, implicit_q=0) as ctx:  # the dense path
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
    assert status == 0 and info["certified"] == 1
    assert cert["eta"] <= 1e-6                                     # Eq. (13)
    s, R, t, p = g["s"], g["R"], g["t"], g["p"]
    # rounded rotations are in SO(3), the anchor is the identity
    assert np.abs(np.einsum("iab,icb->iac", R, R) - np.eye(3)).max() <= 1e-12
    assert np.all(np.linalg.det(R) > 0) and s[0] == 1.0 and np.abs(R[0] - np.eye(3)).max() == 0
    # (a property of the GPU's outputs, evaluated here — not an oracle call)
    # ρ̂ = tr(Q Ūᵀ Ū) equals Eq. (3) at the recovered (s, R, t, p)
    fr, lm, w = sc.frame.astype(np.int64), sc.landmark.astype(np.int64), sc.w
    x = s[fr, None] * np.einsum("eab,eb->ea", R[fr], sc.pts) + t[fr]
    d = x - p[lm]
    rho_edge = float(np.sum(w * np.sum(d * d, axis=1)))
    assert abs(rho_edge - cert["rho_hat"]) <= 1e-8 * (1.0 + abs(rho_edge))
    # Eq. (4): p_k, t_i (i ≥ 1) minimise Eq. (3) at fixed Ū — zero gradients
    res = w[:, None] * d
    gp = np.zeros((sc.M, 3))
    np.add.at(gp, lm, res)
    gt = np.zeros((sc.N, 3))
    np.add.at(gt, fr, res)
    scale = np.abs(res).sum() + 1e-300
    assert np.abs(gp).max() <= 1e-9 * scale
    assert np.abs(gt[1:]).max() <= 1e-9 * scale


# ----------------------------------------------------------------------------- C, D
# The noisy configurations have no known optimum (parity
# unpinned beyond KKT), so GPU-vs-oracle agreement on the same generated input
# is the check: f, X = YYᵀ, λ_min, ρ̂, and the recovered R, s, t, p.
def _end_to_end(xm, sc, opts, Y0=None):
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    st = xo.staircase(dm, xo.Options(**opts), Y0=Y0)
    sol = xo.round_recover(dm, st.Y)
    with xm.Context(profile=1, **opts) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        if Y0 is not None:
            ctx.set_factor(Y0)
        status, info = ctx.solve()
        cert = ctx.certify()
        gsol = ctx.round_recover()
        Yg = ctx.get_factor()
    return dm, st, sol, status, info, cert, gsol, Yg


def _compare(dm, st, sol, status, info, cert, gsol, Yg, xtol=1e-6):
    assert status == 0 and info["certified"] == 1 and st.certified
    assert info["r"] == st.r
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    Xo = st.Y @ st.Y.T
    assert np.linalg.norm(Yg @ Yg.T - Xo) <= xtol * np.linalg.norm(Xo)
    assert abs(cert["lambda_min"] - st.cert.lambda_min) <= 1e-6 * dm.normF
    assert abs(cert["rho_hat"] - sol.rho_hat) <= 1e-8 * (1.0 + abs(sol.rho_hat))
    assert cert["eta"] <= 1e-6
    np.testing.assert_allclose(gsol["s"], sol.s, rtol=xtol, atol=1e-9)
    np.testing.assert_allclose(gsol["R"], sol.R, atol=xtol)
    np.testing.assert_allclose(gsol["t"], sol.t, atol=xtol * max(1.0, np.abs(sol.t).max()))
    ok = np.isfinite(sol.p[:, 0])
    np.testing.assert_allclose(gsol["p"][ok], sol.p[ok], atol=xtol * max(1.0, np.abs(sol.p[ok]).max()))
    assert gsol["n_flipped"] == sol.n_flipped


# Long oracle runs (C: ~3 min, D random init: ~5.5 min of host oracle): run with
# XM_FULL_PARITY=1 (their logs: profiles/r2_full_parity.log); D runs by default.
full_parity = pytest.mark.skipif(not os.environ.get("XM_FULL_PARITY"),
                                 reason="long oracle run: set XM_FULL_PARITY=1")


@pytest.mark.parametrize("cfg", [pytest.param("C", marks=full_parity), "D"])
def test_noisy_configs_end_to_end_vs_oracle(xm, cfg):
    """C is a long noisy forward trajectory with a flat optimum: at the grad
    tolerance 1e-10·‖Q‖_F (reading C8) X is determined only to ~3e-5 — the
    oracle's own X at grad_tol 1e-10 differs from its X at 1e-12 by 2.7e-5
    (1e-11: 3.0e-6; measured, F15's trend) — so C compares X, R, s, t, p at
    1e-4; D (unordered) at the contract's 1e-6."""
    sc = config_scene(cfg)
    opts = dict(rank_cap=5) if cfg == "D" else {}
    _compare(*_end_to_end(xm, sc, opts), xtol=1e-4 if cfg == "C" else 1e-6)


@full_parity
def test_D_random_init_escalates_at_scale(xm):
    """Thm 2/3 at config D's size: a random feasible r = 3 start
    escalates through the staircase (rank cap 5, BASELINE config D) on both
    sides, to the same certified X."""
    from synth.scenes import random_factor
    sc = config_scene("D")
    Y0 = random_factor(sc.N, 3, 4)
    dm, st, sol, status, info, cert, gsol, Yg = _end_to_end(xm, sc, dict(rank_cap=5), Y0=Y0)
    assert len(st.ranks) >= 2 and info["escapes"] >= 1
    _compare(dm, st, sol, status, info, cert, gsol, Yg)


# ----------------------------------------------------------------------------- E, identical Q
def test_E_identical_Q_spmm_and_hvp(xm):
    """Reading C13 at the north-star size: a host-generated symmetric
    30465 × 30465 Q uploaded with xm_set_Q; single products Q·V (r = 1, 3, 4,
    every streaming kernel) and one Riemannian HVP checked on sampled rows /
    frames against numpy on the host, ≤ 1e-12 relative."""
    N = 10155
    n = 3 * N
    rng = np.random.default_rng(77)
    Q = rng.standard_normal((n, n))
    Q += Q.T
    Q *= 0.5
    rows = _sample_rows(N, 16, 5)
    frames = np.unique(rows // 3)                    # includes frame 0 (the anchor)
    for kernel in (0, 1, 2):
        with xm.Context(spmm_kernel=kernel) as ctx:
            ctx.set_Q(Q)
            for r in (1, 3, 4):
                V = rng.standard_normal((n, r))
                out = ctx.spmm(V)
                ref = Q[rows] @ V
                assert rel(out[rows], ref) <= 1e-12, (kernel, r, rel(out[rows], ref))
            if kernel == 0:
                from synth.scenes import random_factor
                r = 3
                Y = random_factor(N, r, 6)
                V = xo.project(Y, rng.standard_normal((n, r)))
                HV = ctx.hvp(Y, V)
                sub = (3 * frames[:, None] + np.arange(3)).ravel()   # block 0 first = anchor
                Ys, Vs = Y[sub], V[sub]
                QYs, QVs = Q[sub] @ Y, Q[sub] @ V
                Lam = xo.multipliers(Ys, QYs)
                ref = xo.project(Ys, 2.0 * QVs - 2.0 * xo.block_apply(Lam, Vs))
                assert rel(HV[sub], ref) <= 1e-12, rel(HV[sub], ref)
    del Q


# ----------------------------------------------------------------------------- matrix-free (NEXT-1)
# The bench headline at E runs the matrix-free products (bench.py --mode auto);
# the same full-size checks through them.
def test_B_implicit_products_and_solve_vs_oracle(xm, B):
    """B matrix-free: Q·V (r = 1, 3, 4, 7) against the oracle's dense Q, and the
    whole solve → certificate → recovery against the oracle's staircase run
    with the same tolerance scale (the shared 16-probe estimate, reading C24)."""
    sc, dm = B
    iq = xo.ImplicitQ(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    est = xo.hutchinson_normF(iq.apply, dm.n)
    st = xo.staircase(dm, normQ=est)
    sol = xo.round_recover(dm, st.Y)
    with xm.Context(implicit_q=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        for r in (1, 3, 4, 7):
            V = random_tangent_ambient(sc.N, r, 30 + r)
            assert rel(ctx.spmm(V), dm.Q @ V) <= 1e-10, r
        status, info = ctx.solve()
        cert = ctx.certify()
        gsol = ctx.round_recover()
        Yg = ctx.get_factor()
    assert abs(info["normQ"] - est) <= 1e-10 * est
    assert status == 0 and info["certified"] == 1 and st.certified
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    Xo = st.Y @ st.Y.T
    assert np.linalg.norm(Yg @ Yg.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
    assert cert["eta"] <= 1e-6
    np.testing.assert_allclose(gsol["s"], sol.s, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(gsol["R"], sol.R, atol=1e-6)
    np.testing.assert_allclose(gsol["t"], sol.t, atol=1e-6 * max(1.0, np.abs(sol.t).max()))


def test_E_implicit_noisy_sampled_rows_certified_and_optimal(xm, E_noisy):
    """E with noise through the matrix-free products (the headline mode): sampled
    rows of Q·V against the oracle's row-wise Schur complement (reading C13
    tolerance), a certified zero duality gap, Eq. (3) at the recovered
    (s, R, t, p) = ρ̂, and first-order optimality of the recovered t, p."""
    sc = E_noisy
    rows = _sample_rows(sc.N, 12, 5)
    info_q = {}
    QI = xo.q_rows(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w, rows, info=info_q)
    tol = max(1e-10, 8 * np.finfo(float).eps * info_q["kappa_K"] * info_q["S_I_norm"]
              / np.linalg.norm(QI))
    with xm.Context(implicit_q=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        for r in (1, 3, 4):
            V = random_tangent_ambient(sc.N, r, 41 + r)
            assert rel(ctx.spmm(V)[rows], QI @ V) <= tol, r
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
    assert status == 0 and info["certified"] == 1
    assert cert["eta"] <= 1e-6
    s, R, t, p = g["s"], g["R"], g["t"], g["p"]
    assert np.abs(np.einsum("iab,icb->iac", R, R) - np.eye(3)).max() <= 1e-12
    assert np.all(np.linalg.det(R) > 0) and s[0] == 1.0
    fr, lm, w = sc.frame.astype(np.int64), sc.landmark.astype(np.int64), sc.w
    x = s[fr, None] * np.einsum("eab,eb->ea", R[fr], sc.pts) + t[fr]
    d = x - p[lm]
    rho_edge = float(np.sum(w * np.sum(d * d, axis=1)))
    assert abs(rho_edge - cert["rho_hat"]) <= 1e-8 * (1.0 + abs(rho_edge))
    res = w[:, None] * d
    gp = np.zeros((sc.M, 3))
    np.add.at(gp, lm, res)
    gt = np.zeros((sc.N, 3))
    np.add.at(gt, fr, res)
    scale = np.abs(res).sum() + 1e-300
    assert np.abs(gp).max() <= 1e-9 * scale
    assert np.abs(gt[1:]).max() <= 1e-9 * scale
