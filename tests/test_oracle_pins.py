"""Pins for the CPU oracle (oracle/xm_oracle.py) against what the paper and the
mathematics fix — never against the oracle's own formulas.

Each test names the passage it pins.  Brute-force references here (dense least
squares over (t, p), dense eigendecomposition, the paper's printed B¹..B⁵,
Umeyama's closed form, finite differences) are independent of the oracle's
Schur-complement / projection formulas, so a dropped term, a wrong sign or a
transposed operand in the oracle fails one of them.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import make_scene, random_factor, random_tangent_ambient

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def gt_factor(sc):
    """Y_gt = [s_0R_0, …]ᵀ stacked: Y_i = (s_i R_i)ᵀ."""
    return np.concatenate([(sc.s[i] * sc.R[i]).T for i in range(sc.N)], axis=0)


def brute_marginal_objective(sc, Y):
    """min_{t (t_0=0), p} Σ_e w_e‖Y_iᵀũ_e + t_i − p_k‖² by dense weighted least
    squares, one coordinate at a time (Eq. (3) P:104-109 at fixed U; the
    SPEC's marginal_objective_oracle S:151-159)."""
    N, M = sc.N, sc.M
    E = len(sc.frame)
    r = Y.shape[1]
    A = np.zeros((E, (N - 1) + M))
    for e in range(E):
        i, k = sc.frame[e], sc.landmark[e]
        if i >= 1:
            A[e, i - 1] = 1.0
        A[e, (N - 1) + k] = -1.0
    sw = np.sqrt(sc.w)
    total = 0.0
    for c in range(r):
        b = np.array([Y[3 * sc.frame[e]:3 * sc.frame[e] + 3, c] @ sc.pts[e] for e in range(E)])
        x, *_ = np.linalg.lstsq(sw[:, None] * A, -sw * b, rcond=None)
        res = A @ x + b
        total += float(np.sum(sc.w * res * res))
    return total


# ----------------------------------------------------------------------------- Q
def test_golden_laplacian_two_frames_one_landmark():
    g = GOLD["laplacian_2frames_1landmark"]
    pts = np.array([[0.1, 0.2, 1.0], [0.3, -0.1, 2.0]])
    H = xo.quadratic_form(2, 1, np.array([0, 1]), np.array([0, 0]), pts, np.ones(2)).toarray()
    Qtp = H[6:, 6:]                                  # (t_0, t_1, p_0) block
    np.testing.assert_array_equal(Qtp, np.array(g["Q_tp"], float))


def test_golden_two_edges_one_frame_degree():
    g = GOLD["two_edges_one_frame"]
    pts = np.array([[0.1, 0.2, 1.0], [0.3, -0.1, 2.0]])
    H = xo.quadratic_form(1, 2, np.array([0, 0]), np.array([0, 1]), pts, np.array(g["weights"])).toarray()
    assert H[3, 3] == g["Q2"]                       # t_0 diagonal = weighted degree


def test_laplacian_rows_sum_to_zero_and_degrees():
    """Q_tp·1 = 0, diag(Q_2)=frame degrees, diag(Q_3)=landmark degrees."""
    sc = make_scene(6, 40, "unordered", seed=3, vis_prob=0.5, weights="uniform")
    H = xo.quadratic_form(sc.N, sc.M, sc.frame.astype(int), sc.landmark.astype(int), sc.pts, sc.w).toarray()
    n = 3 * sc.N
    Qtp = H[n:, n:]
    assert np.abs(Qtp @ np.ones(sc.N + sc.M)).max() < 1e-12
    np.testing.assert_allclose(np.diag(Qtp)[:sc.N], np.bincount(sc.frame, sc.w, sc.N), rtol=1e-15)
    np.testing.assert_allclose(np.diag(Qtp)[sc.N:], np.bincount(sc.landmark, sc.w, sc.M), rtol=1e-15)
    # single edge U-U block = w ũ ũᵀ
    H1 = xo.quadratic_form(1, 1, np.array([0]), np.array([0]), np.array([[0.3, -0.2, 1.5]]), np.array([2.0])).toarray()
    v = np.array([0.3, -0.2, 1.5])
    np.testing.assert_allclose(H1[:3, :3], 2.0 * np.outer(v, v), rtol=1e-15)


@pytest.mark.parametrize("seed", range(6))
def test_prop1_equivalence_brute_force(seed):
    """Prop. 1, acceptance 1: tr(QUᵀU) = min_{t,p} Eq.(3)."""
    rng = np.random.default_rng(seed)
    N = int(rng.integers(2, 8))
    M = int(rng.integers(5, 30))
    sc = make_scene(N, M, "unordered", seed=seed, vis_prob=0.5, weights="uniform",
                    sigma_d=0.1, sigma_u=0.01)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    for r in (3, 4, 5):
        Y = random_factor(N, r, seed * 10 + r, anchor_identity=(r == 3))
        f_q = float(np.vdot(Y, dm.Q @ Y))
        f_b = brute_marginal_objective(sc, Y)
        assert abs(f_q - f_b) <= 1e-9 * max(1.0, abs(f_b)), (r, f_q, f_b)


@pytest.mark.parametrize("cfg", [
    dict(N=9, M=120, kind="unordered", vis_prob=0.5, sigma_d=0.1, sigma_u=0.01),
    dict(N=30, M=400, kind="loop", window=5, sigma_d=0.05),
    dict(N=25, M=500, kind="road", track_mean=5.0, sigma_u=1e-3, sigma_d=0.01, weights="uniform"),
    dict(N=1, M=6, kind="unordered", vis_prob=1.0),
], ids=lambda c: f"{c['kind']}{c['N']}")
def test_q_rows_matches_dense_Q(cfg):
    """Sampled-row Schur complement (q_rows) = rows of the dense build_Q — the
    latter pinned above by Prop. 1 brute force; incl. the first / last row,
    duplicate observations and N = 1 (Q = 0)."""
    sc = make_scene(seed=4, **cfg)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    n = 3 * sc.N
    rows = np.unique(np.concatenate([[0, n - 1], np.random.default_rng(1).integers(0, n, 7)]))
    fr = np.concatenate([sc.frame, sc.frame[:3]])         # duplicates: keep first
    lm = np.concatenate([sc.landmark, sc.landmark[:3]])
    pts = np.concatenate([sc.pts, 2.0 * sc.pts[:3]])
    w = np.concatenate([sc.w, sc.w[:3]])
    QI = xo.q_rows(sc.N, sc.M, fr, lm, pts, w, rows)
    assert QI.shape == (rows.size, n)
    assert np.linalg.norm(QI - dm.Q[rows]) <= 1e-12 * max(1.0, dm.normF)


def test_q_rows_noise_free_annihilates_ground_truth():
    """F1: Q[I,:] Y_gt = 0 on a noise-free scene, every row."""
    sc = make_scene(15, 300, "unordered", seed=2, vis_prob=0.4)
    QI = xo.q_rows(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w, np.arange(3 * sc.N))
    assert np.linalg.norm(QI @ gt_factor(sc)) <= 1e-10 * np.linalg.norm(QI)
    assert np.linalg.norm(QI - QI.T) <= 1e-12 * np.linalg.norm(QI)


def test_edge_objective_brute_force_and_ground_truth():
    """Eq. (3): zero at the noise-free ground truth, and equal to a
    per-observation loop at arbitrary (s, R, t, p)."""
    sc = make_scene(6, 40, "unordered", seed=3, vis_prob=0.6)
    assert xo.edge_objective(sc.frame, sc.landmark, sc.pts, sc.w, sc.s, sc.R, sc.t, sc.p) \
        <= 1e-20 * len(sc.frame) + 1e-24
    rng = np.random.default_rng(0)
    s = rng.uniform(0.5, 2.0, sc.N)
    R = np.stack([np.linalg.qr(rng.standard_normal((3, 3)))[0] for _ in range(sc.N)])
    t = rng.standard_normal((sc.N, 3))
    p = rng.standard_normal((sc.M, 3))
    tot = 0.0
    for e in range(len(sc.frame)):
        i, k = int(sc.frame[e]), int(sc.landmark[e])
        d = s[i] * (R[i] @ sc.pts[e]) + t[i] - p[k]
        tot += sc.w[e] * float(d @ d)
    assert abs(xo.edge_objective(sc.frame, sc.landmark, sc.pts, sc.w, s, R, t, p) - tot) \
        <= 1e-12 * tot


def test_N1_gives_zero_Q():
    """N = 1 ⇒ Q = 0."""
    sc = make_scene(1, 7, "unordered", seed=0, vis_prob=1.0)
    dm = xo.build_Q(1, 7, sc.frame, sc.landmark, sc.pts, sc.w)
    assert np.abs(dm.Q).max() < 1e-13


def test_noise_free_null_space_is_ground_truth():
    """F1 / S:149: noise-free ⇒ Q ⪰ 0, 3-dim null space spanned by Y_gt, f(Y_gt)=0."""
    sc = make_scene(12, 200, "unordered", seed=1, vis_prob=0.4)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    ev = np.linalg.eigvalsh(dm.Q)
    nQ = dm.normF
    assert ev[0] >= -1e-9 * nQ
    assert np.all(np.abs(ev[:3]) <= 1e-10 * nQ) and ev[3] > 1e-3 * nQ
    Yg = gt_factor(sc)
    assert np.linalg.norm(dm.Q @ Yg) <= 1e-10 * nQ
    # Q symmetric
    assert np.abs(dm.Q - dm.Q.T).max() <= 1e-12 * nQ


def test_anchor_independence_and_singletons():
    """F2 (reading C2): grounding another translation gives the same Q;
    F10: singleton landmarks do not change Q."""
    sc = make_scene(5, 30, "unordered", seed=4, vis_prob=0.5, sigma_d=0.2, weights="uniform")
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    H = xo.quadratic_form(sc.N, sc.M, sc.frame.astype(int), sc.landmark.astype(int), sc.pts, sc.w).toarray()
    n = 3 * sc.N
    for ground in (2, 4):
        keep = [j for j in range(n, n + sc.N + sc.M) if j != n + ground]
        Huu, Hux, Hxx = H[:n, :n], H[:n, keep], H[np.ix_(keep, keep)]
        Qg = Huu - Hux @ np.linalg.solve(Hxx, Hux.T)
        np.testing.assert_allclose(Qg, dm.Q, atol=1e-10 * dm.normF)
    # add two singleton landmarks
    fr = np.concatenate([sc.frame, [1, 3]])
    lm = np.concatenate([sc.landmark, [sc.M, sc.M + 1]])
    pts = np.concatenate([sc.pts, [[0.1, 0.2, 3.0], [-0.3, 0.1, 5.0]]])
    w = np.concatenate([sc.w, [0.7, 0.9]])
    dm2 = xo.build_Q(sc.N, sc.M + 2, fr, lm, pts, w)
    np.testing.assert_allclose(dm2.Q, dm.Q, atol=1e-12 * dm.normF)


def test_gauge_invariance():
    """f(Y O) = f(Y) for orthogonal O (r×r)."""
    sc = make_scene(6, 40, "unordered", seed=5, vis_prob=0.5, sigma_d=0.1)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    Y = random_factor(sc.N, 4, 2)
    O, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((4, 4)))
    assert abs(xo.cost(dm.Q, Y @ O) - xo.cost(dm.Q, Y)) <= 1e-12 * abs(xo.cost(dm.Q, Y))


def test_s_pattern_matches_numeric_structure():
    """H3 pattern = nonzero 3×3 block structure of S (random weights ⇒ no
    accidental cancellation)."""
    sc = make_scene(15, 60, "loop", seed=2, window=4)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    rowptr, colidx = xo.s_pattern(sc.N, sc.frame, sc.landmark)
    blk = np.abs(dm.S).reshape(sc.N, 3, sc.N, 3).max(axis=(1, 3)) > 0
    for i in range(sc.N):
        np.testing.assert_array_equal(colidx[rowptr[i]:rowptr[i + 1]], np.nonzero(blk[i])[0])
    # Q itself is block-dense for a connected graph (F1)
    qblk = np.abs(dm.Q).reshape(sc.N, 3, sc.N, 3).max(axis=(1, 3)) > 0
    assert qblk.all()


# --------------------------------------------------------------------- manifold
@pytest.fixture(scope="module")
def small_problem():
    sc = make_scene(7, 60, "unordered", seed=11, vis_prob=0.5, sigma_d=0.2, sigma_u=0.01)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    return sc, dm


@pytest.mark.parametrize("r", [3, 4, 5])
def test_projection_properties(small_problem, r):
    """Tangent space of {Y_0Y_0ᵀ = I, Y_iY_iᵀ = α_iI}: the derivative
    of the constraints gives sym(V_0Y_0ᵀ) = 0, sym₀(V_iY_iᵀ) = 0; projection is
    idempotent, self-adjoint, and the radial direction is kept."""
    sc, dm = small_problem
    Y = random_factor(sc.N, r, 7)
    A = random_tangent_ambient(sc.N, r, 1)
    B = random_tangent_ambient(sc.N, r, 2)
    V = xo.project(Y, A)
    for i in range(sc.N):
        M_ = V[3 * i:3 * i + 3] @ Y[3 * i:3 * i + 3].T
        Ms = 0.5 * (M_ + M_.T)
        if i == 0:
            assert np.abs(Ms).max() < 1e-12
        else:
            assert np.abs(Ms - np.trace(Ms) / 3 * np.eye(3)).max() < 1e-12
        # normal component = (traceless) symmetric × Y_i
        Nn = (A - V)[3 * i:3 * i + 3] @ Y[3 * i:3 * i + 3].T
        assert np.abs(Nn - Nn.T).max() < 1e-10
        if i > 0:
            assert abs(np.trace(Nn)) < 1e-10
    np.testing.assert_allclose(xo.project(Y, V), V, atol=1e-12)
    assert abs(np.vdot(xo.project(Y, A), B) - np.vdot(A, xo.project(Y, B))) < 1e-10
    PY = xo.project(Y, Y)
    np.testing.assert_allclose(PY[3:], Y[3:], atol=1e-12)
    assert np.abs(PY[:3]).max() < 1e-12


def test_multipliers_match_paper_B_matrices(small_problem):
    """Λ_i solves (QY)_i ≈ (Σ_ℓ y_ℓ B^ℓ) Y_i in least squares with the B¹..B⁵
    printed in App. A.4 — 5 unknowns per block; anchor: 6."""
    sc, dm = small_problem
    Y = random_factor(sc.N, 4, 3)
    QY = dm.Q @ Y
    Lam = xo.multipliers(Y, QY)
    Bs = [np.array([[1, 0, 0], [0, -1, 0], [0, 0, 0]]), np.array([[0, 0, 0], [0, 1, 0], [0, 0, -1]]),
          np.array([[0, 1, 0], [1, 0, 0], [0, 0, 0]]), np.array([[0, 0, 1], [0, 0, 0], [1, 0, 0]]),
          np.array([[0, 0, 0], [0, 0, 1], [0, 1, 0]])]
    E6 = [np.diag([1.0, 0, 0]), np.diag([0, 1.0, 0]), np.diag([0, 0, 1.0])] + Bs[2:]
    for i in range(sc.N):
        Yi, Gi = Y[3 * i:3 * i + 3], QY[3 * i:3 * i + 3]
        basis = E6 if i == 0 else Bs
        Amat = np.stack([(Bl @ Yi).ravel() for Bl in basis], axis=1)
        y, *_ = np.linalg.lstsq(Amat, Gi.ravel(), rcond=None)
        Lref = sum(c * Bl for c, Bl in zip(y, basis))
        np.testing.assert_allclose(Lam[i], Lref, atol=1e-9 * np.abs(Lref).max() + 1e-12)


def test_licq_rank(small_problem):
    """App. A.4 / S:406: {A_i Uᵀ} has rank m = 5N+1 at feasible points (N ≤ 6)."""
    N = 5
    Y = random_factor(N, 4, 9)
    n = 3 * N
    Bs = [np.array([[1, 0, 0], [0, -1, 0], [0, 0, 0]]), np.array([[0, 0, 0], [0, 1, 0], [0, 0, -1]]),
          np.array([[0, 1, 0], [1, 0, 0], [0, 0, 0]]), np.array([[0, 0, 1], [0, 0, 0], [1, 0, 0]]),
          np.array([[0, 0, 0], [0, 0, 1], [0, 1, 0]])]
    E6 = [np.diag([1.0, 0, 0]), np.diag([0, 1.0, 0]), np.diag([0, 0, 1.0])] + Bs[2:]
    cols = []
    for i in range(N):
        for Bl in (E6 if i == 0 else Bs):
            A = np.zeros((n, n))
            A[3 * i:3 * i + 3, 3 * i:3 * i + 3] = Bl
            cols.append((A @ Y).ravel())
    assert np.linalg.matrix_rank(np.stack(cols, 1)) == 5 * N + 1


def test_retraction_properties(small_problem):
    """step 0 ⇒ identity; feasibility; ‖R(hV) − (Y+hV)‖ = O(h²)."""
    sc, _ = small_problem
    Y = random_factor(sc.N, 5, 4)
    V = xo.project(Y, random_tangent_ambient(sc.N, 5, 5))
    np.testing.assert_allclose(xo.retract(Y, 0 * V), Y, atol=1e-14)
    errs = []
    for h in (1e-3, 5e-4, 2.5e-4, 1.25e-4):
        Yh = xo.retract(Y, h * V)
        errs.append(np.linalg.norm(Yh - (Y + h * V)))
        B = xo.blocks(Yh)
        G = np.einsum("iar,ibr->iab", B, B)
        np.testing.assert_allclose(G[0], np.eye(3), atol=1e-12)
        a = np.trace(G, axis1=1, axis2=2) / 3
        assert np.abs(G - a[:, None, None] * np.eye(3)).max() < 1e-12
    ratios = [errs[j] / errs[j + 1] for j in range(3)]
    assert all(3.6 < q < 4.4 for q in ratios), ratios


@pytest.mark.parametrize("r", [3, 4, 5])
def test_gradient_finite_differences(small_problem, r):
    """S:241, acceptance 4: d/dh f(R(hV)) at 0 = ⟨grad f, V⟩."""
    sc, dm = small_problem
    Y = random_factor(sc.N, r, 20 + r)
    V = xo.project(Y, random_tangent_ambient(sc.N, r, 30 + r))
    g, _ = xo.rgrad(Y, dm.Q @ Y)
    h = 1e-5
    fd = (xo.cost(dm.Q, xo.retract(Y, h * V)) - xo.cost(dm.Q, xo.retract(Y, -h * V))) / (2 * h)
    assert abs(fd - np.vdot(g, V)) <= 1e-6 * max(1.0, abs(fd))
    # Euclidean gradient 2QY vs FD of the ambient cost
    A = random_tangent_ambient(sc.N, r, 40 + r)
    fdE = (xo.cost(dm.Q, Y + h * A) - xo.cost(dm.Q, Y - h * A)) / (2 * h)
    assert abs(fdE - np.vdot(2 * dm.Q @ Y, A)) <= 1e-6 * max(1.0, abs(fdE))


@pytest.mark.parametrize("r", [3, 4, 5])
def test_hessian_finite_differences_and_symmetry(small_problem, r):
    """S:258-259, acceptance 4: Hess[V] = P_Y(D grad[V]) (FD of the smoothly
    extended gradient), self-adjoint."""
    sc, dm = small_problem
    Y = random_factor(sc.N, r, 50 + r)
    V = xo.project(Y, random_tangent_ambient(sc.N, r, 60 + r))
    W = xo.project(Y, random_tangent_ambient(sc.N, r, 70 + r))
    _, Lam = xo.rgrad(Y, dm.Q @ Y)
    HV = xo.hess(dm.Q, Y, Lam, V)
    h = 1e-6
    gp, _ = xo.rgrad(Y + h * V, dm.Q @ (Y + h * V))
    gm, _ = xo.rgrad(Y - h * V, dm.Q @ (Y - h * V))
    fd = xo.project(Y, (gp - gm) / (2 * h))
    assert np.linalg.norm(fd - HV) <= 1e-5 * np.linalg.norm(HV)
    HW = xo.hess(dm.Q, Y, Lam, W)
    assert abs(np.vdot(HV, W) - np.vdot(V, HW)) <= 1e-10 * np.linalg.norm(HV) * np.linalg.norm(W)


# ------------------------------------------------------------------ certificate
def test_golden_min_eig_diag():
    g = GOLD["min_eig_diag"]
    Z = np.diag(g["Z_diag"])
    lam, v = xo.dense_min_eig(Z)
    assert lam == g["lambda_min"]
    np.testing.assert_allclose(v, g["v"], atol=0)
    lam2, v2, _, _ = xo.lanczos_min_eig(lambda x: Z @ x, 3, 1e-12)
    assert abs(lam2 - g["lambda_min"]) < 1e-12
    np.testing.assert_allclose(np.abs(v2), g["v"], atol=1e-10)


def test_lanczos_matches_dense_eig(small_problem):
    sc, dm = small_problem
    Y = random_factor(sc.N, 4, 13)
    _, Lam = xo.rgrad(Y, dm.Q @ Y)
    Z = xo.z_matrix(dm.Q, Lam)
    lam_d = np.linalg.eigvalsh(Z)[0]
    lam_l, v, k, res = xo.lanczos_min_eig(lambda x: Z @ x, Z.shape[0], 1e-10 * dm.normF)
    assert abs(lam_l - lam_d) <= 1e-9 * dm.normF
    assert np.linalg.norm(Z @ v - lam_l * v) <= 1e-8 * dm.normF


def test_golden_suboptimality_and_bound():
    for c in GOLD["suboptimality"]["cases"]:
        assert xo.suboptimality(c["rho_hat"], c["rho_lower"]) == c["eta"]
    for c in GOLD["rigorous_lower_bound"]["cases"]:
        cert = xo.Certificate(lambda_min=c["lambda_min"], v=None, rho_dual=c["rho_dual"], Lam=None,
                              kkt_resid=0, grad_norm=0, lanczos_steps=0, trace_X=c["trace_X"])
        rep = xo.report(cert, 0.0)
        lowE = max(0.0, c["lambda_min"]) * c["trace_X"] + c["rho_dual"]
        assert lowE == c["lower"]
        assert abs(rep["eta_E"] - (0.0 - lowE) / (1 + abs(lowE))) < 1e-15


# ------------------------------------------------------------------ staircase
def test_noise_free_tight_certified_and_gt_recovered():
    """Acceptance 2: noise-free ⇒ certified at
    r=3, f≈0, λ_min ≥ −1e-6‖Q‖, η ≤ 1e-6, recovered poses = GT, no flips."""
    sc = make_scene(20, 100, "unordered", seed=2, vis_prob=0.4)
    dm, st, sol, rep = xo.solve(sc)
    nQ = dm.normF
    assert st.certified and st.r == 3
    assert abs(st.f) <= 1e-10 * nQ
    assert st.cert.lambda_min >= -1e-6 * nQ
    assert rep["eta"] <= 1e-6
    np.testing.assert_allclose(sol.s, sc.s, atol=1e-8)
    np.testing.assert_allclose(sol.R, sc.R, atol=1e-8)
    np.testing.assert_allclose(sol.t, sc.t, atol=1e-7)
    np.testing.assert_allclose(sol.p, sc.p, atol=1e-7)
    assert sol.n_flipped == 0
    # KKT: ‖ZY‖ ≤ 1e-8‖Q‖; multipliers vanish; f = tr Λ₀ (F5)
    assert st.cert.kkt_resid <= 1e-8 * nQ
    assert np.abs(st.cert.Lam).max() <= 1e-8 * nQ
    # Lanczos vs dense brute force on the same Z
    lam_d, _ = xo.dense_min_eig(xo.z_matrix(dm.Q, st.cert.Lam))
    assert abs(lam_d - st.cert.lambda_min) <= 1e-7 * nQ


def test_noisy_kkt_identities():
    """F5 / Thm 1: at a certified critical point f = tr Λ₀ = ρ_dual,
    ⟨(QY)_i, Y_i⟩ ≈ 0 (i ≥ 1), ⟨V,HessV⟩ = 2⟨V,ZV⟩; edge objective (Eq. (3))
    at the recovered solution = f(Ŷ) (Prop. 1)."""
    sc = make_scene(8, 80, "unordered", seed=7, vis_prob=0.5, sigma_d=0.1, sigma_u=0.01, weights="uniform")
    dm, st, sol, rep = xo.solve(sc)
    nQ = dm.normF
    assert st.certified
    assert abs(st.f - st.cert.rho_dual) <= 1e-8 * max(1.0, abs(st.f))
    B, G = xo.blocks(st.Y), xo.blocks(st.QY)
    assert np.abs(np.einsum("iar,iar->i", B, G)[1:]).max() <= 1e-8 * nQ
    V = xo.project(st.Y, random_tangent_ambient(sc.N, st.r, 3))
    HV = xo.hess(dm.Q, st.Y, st.cert.Lam, V)
    Z = xo.z_matrix(dm.Q, st.cert.Lam)
    assert abs(np.vdot(V, HV) - 2 * np.vdot(V, Z @ V)) <= 1e-7 * abs(np.vdot(V, HV))
    assert abs(sol.edge_objective - sol.rho_hat) <= 1e-8 * max(1.0, abs(sol.rho_hat))
    assert rep["eta"] <= 1e-6


def test_non_tight_instance_chain_inequality():
    """Eq. (14): on a high-noise instance the relaxation is
    not tight (rank 4 certified optimum, det flips); still ρ_lower ≤ ρ̂ and
    η > 0, and the certified SDP value f ≤ ρ̂."""
    sc = make_scene(8, 80, "unordered", seed=7, vis_prob=0.5, sigma_d=0.3, sigma_u=0.01, weights="uniform")
    dm, st, sol, rep = xo.solve(sc)
    assert st.certified and st.r == 4
    assert rep["rho_lower"] <= sol.rho_hat + 1e-9 * (1 + abs(sol.rho_hat))
    assert st.f <= sol.rho_hat and rep["eta"] > 1e-6


def test_random_init_escalates_and_reaches_same_X():
    """Thm 2/3, Fig. 8 behaviour, acceptance 7; F6: random
    init at r=3 stalls at a spurious critical point, the escape along [0, v]
    lifts to r=4 and the staircase certifies the same X as identity init."""
    sc = make_scene(10, 500, "unordered", seed=0, vis_prob=0.6)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    st_id = xo.staircase(dm)
    st_rd = xo.staircase(dm, Y0=random_factor(sc.N, 3, 1))
    assert st_rd.ranks == [3, 4] and st_rd.certified
    Xa = st_id.Y @ st_id.Y.T
    Xb = st_rd.Y @ st_rd.Y.T
    assert np.linalg.norm(Xa - Xb) <= 1e-8 * np.linalg.norm(Xa)


def test_escape_direction_is_tangent_and_descends():
    """Thm 2: D = [0, v] is tangent at [Y, 0]; line search lowers f."""
    sc = make_scene(10, 500, "unordered", seed=0, vis_prob=0.6)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    opts = xo.Options(rank_cap=3)
    st = xo.staircase(dm, opts, Y0=random_factor(sc.N, 3, 1))
    assert st.cert.lambda_min < 0 and not st.certified
    Yz = np.concatenate([st.Y, np.zeros((st.Y.shape[0], 1))], 1)
    D = np.zeros_like(Yz)
    D[:, 3] = st.cert.v
    np.testing.assert_allclose(xo.project(Yz, D), D, atol=1e-12)
    Yp, alpha, df = xo.escape(dm.Q, st.Y, st.QY, st.cert.v)
    assert df < 0 and xo.cost(dm.Q, Yp) < st.f


# -------------------------------------------------------------- N = 2 closed form
def umeyama(x, y, c):
    """Weighted similarity registration y ≈ sRx + t (Umeyama 1991)."""
    cs = c / c.sum()
    mx, my = cs @ x, cs @ y
    xc, yc = x - mx, y - my
    Sxy = (cs[:, None] * yc).T @ xc
    U, D, Vt = np.linalg.svd(Sxy)
    Sg = np.diag([1.0, 1.0, np.sign(np.linalg.det(U) * np.linalg.det(Vt))])
    R = U @ Sg @ Vt
    var = float(np.sum(cs * np.sum(xc * xc, 1)))
    s = float(np.trace(np.diag(D) @ Sg)) / var
    return s, R, my - s * R @ mx


@pytest.mark.parametrize("seed", range(4))
def test_two_frames_equal_umeyama(seed):
    """Remark 1, acceptance 3: N = 2 SBA = scaled point cloud
    registration; eliminating p_k gives weights c_k = w_0k w_1k/(w_0k + w_1k)."""
    sc = make_scene(2, 40, "unordered", seed=seed, vis_prob=0.9, sigma_d=0.05, sigma_u=0.01,
                    weights="uniform")
    dm, st, sol, rep = xo.solve(sc)
    assert st.certified
    idx0 = {k: e for e, (i, k) in enumerate(zip(sc.frame, sc.landmark)) if i == 0}
    idx1 = {k: e for e, (i, k) in enumerate(zip(sc.frame, sc.landmark)) if i == 1}
    both = sorted(set(idx0) & set(idx1))
    x = np.array([sc.pts[idx1[k]] for k in both])
    y = np.array([sc.pts[idx0[k]] for k in both])
    w0 = np.array([sc.w[idx0[k]] for k in both])
    w1 = np.array([sc.w[idx1[k]] for k in both])
    s, R, t = umeyama(x, y, w0 * w1 / (w0 + w1))
    assert abs(sol.s[1] - s) <= 1e-8 * s
    ang = math.atan2(np.linalg.norm(R.T @ sol.R[1] - sol.R[1].T @ R) / math.sqrt(2),
                     np.trace(R.T @ sol.R[1]) - 1)
    assert abs(ang) <= 1e-6
    np.testing.assert_allclose(sol.t[1], t, atol=1e-7 * max(1.0, np.abs(t).max()))


# ------------------------------------------------------------------ validation
def test_validation_errors():
    fr = np.array([0, 1, 0, 1])
    lm = np.array([0, 0, 1, 1])
    pts = np.array([[0.1, 0.1, 1.0]] * 4)
    with pytest.raises(xo.OracleError) as e:
        xo.validate(2, 2, np.array([0, 2, 0, 1]), lm, pts)
    assert e.value.code == "EINVAL"
    bad = pts.copy()
    bad[2, 2] = -1.0
    with pytest.raises(xo.OracleError):
        xo.validate(2, 2, fr, lm, bad)
    with pytest.raises(xo.OracleError):
        xo.validate(2, 2, fr, lm, pts, np.array([1.0, 0.0, 1.0, 1.0]))
    nan = pts.copy()
    nan[0, 0] = np.nan
    with pytest.raises(xo.OracleError):
        xo.validate(2, 2, fr, lm, nan)
    # disconnected: two frames, private landmarks
    with pytest.raises(xo.OracleError) as e:
        xo.validate(2, 2, np.array([0, 1]), np.array([0, 1]), pts[:2])
    assert e.value.code == "EDISCONNECTED"
    # duplicates: keep first
    f2 = np.array([0, 1, 0, 1, 0])
    l2 = np.array([0, 0, 1, 1, 0])
    p2 = np.concatenate([pts, [[9.0, 9.0, 9.0]]])
    out = xo.validate(2, 2, f2, l2, p2)
    assert out[4] == 1 and len(out[0]) == 4 and not np.any(out[2][:, 0] == 9.0)


# ---------------------------------------------------------------------------
# XM² (S:472-476 edge_residuals, S:533-537 xm_squared; reading C22)
# ---------------------------------------------------------------------------

def _rot_err(R, Rg):
    """Geodesic angle via atan2 (F12 practical note)."""
    M = R.transpose(0, 2, 1) @ Rg
    sk = M - M.transpose(0, 2, 1)
    sn = np.linalg.norm(sk, axis=(1, 2)) / math.sqrt(2)
    return np.arctan2(sn, np.trace(M, axis1=1, axis2=2) - 1.0)


def test_edge_residuals_sum_to_eq3_and_are_linear_in_w():
    """Σ residuals = Eq. (3) at the solution, here evaluated by the
    brute-force marginal least squares (independent of the oracle's recovery);
    S:478: doubling one weight doubles that residual only."""
    sc = make_scene(8, 120, "unordered", seed=5, vis_prob=0.6, sigma_u=1e-2, sigma_d=0.05)
    dm, st, sol, rep = xo.solve(sc)
    res = xo.edge_residuals(sc.frame, sc.landmark, sc.pts, sc.w, sol)
    assert np.all(res >= 0)
    brute = brute_marginal_objective(sc, sol.Yr)     # min over (t, p) at the rounded U
    assert abs(res.sum() - brute) <= 1e-9 * (1 + brute)
    w2 = sc.w.copy()
    w2[7] *= 2.0
    res2 = xo.edge_residuals(sc.frame, sc.landmark, sc.pts, w2, sol)
    assert res2[7] == pytest.approx(2 * res[7], rel=1e-14)
    assert np.array_equal(np.delete(res2, 7), np.delete(res, 7))


def test_xm2_select_count_and_order():
    """10 edges → exactly ⌊0.1·10⌋ = 1 dropped, the largest residual;
    ties broken by (landmark, frame) ascending (C22)."""
    N, M = 2, 5
    fr = np.array([0, 1] * 5)
    lm = np.repeat(np.arange(5), 2)
    res = np.array([1.0, 2, 3, 4, 5, 6, 7, 9, 8, 0.5])
    keep = xo.xm2_select(N, M, fr, lm, res, 0.1)
    assert (~keep).sum() == 1 and not keep[7]
    res_tie = np.array([9.0, 1, 1, 1, 9, 1, 1, 1, 1, 1])  # edges 0 (lm 0) and 4 (lm 2) tie
    keep = xo.xm2_select(N, M, fr, lm, res_tie, 0.1)
    assert not keep[0] and keep[4]
    E = 37
    rng = np.random.default_rng(0)
    fr = np.concatenate([np.zeros(20, int), np.ones(17, int)])
    lm = np.concatenate([np.arange(20), np.arange(17)])   # landmarks 0..16 seen by both frames
    keep = xo.xm2_select(2, 20, fr, lm, rng.uniform(size=E), 0.1)
    assert (~keep).sum() == math.floor(0.1 * E)


def test_xm2_select_restores_minimal_bridges():
    """S:536/S:562 never disconnect: in a chain of 4 frames joined by single
    landmarks, dropping the top residuals would cut bridges; exactly the
    bridges needed to reconnect are restored, smallest residual first."""
    # frames 0-1 share landmark 0; 1-2 share landmark 1; 2-3 share landmark 2;
    # each frame also sees 4 private landmarks (3..18)
    fr, lm = [], []
    for i, k in [(0, 0), (1, 0), (1, 1), (2, 1), (2, 2), (3, 2)]:
        fr.append(i), lm.append(k)
    for i in range(4):
        for q in range(4):
            fr.append(i), lm.append(3 + 4 * i + q)
    fr, lm = np.array(fr), np.array(lm)
    E = len(fr)                                      # 22 → ⌊2.2⌋ = 2 dropped
    res = np.ones(E)
    res[1], res[3] = 10.0, 20.0                      # (1,0) and (2,1): both bridge edges
    keep = xo.xm2_select(4, 19, fr, lm, res, 0.1)
    assert keep[1] and keep[3]                       # both had to come back
    assert xo.connected_components(4, 19, fr[keep], lm[keep]) == 1
    res[5] = 15.0                                    # a third candidate: (3,2), also a bridge
    keep = xo.xm2_select(4, 19, fr, lm, res, 0.1)    # drops (2,1) and (3,2); both restored
    assert keep.all()


def test_xm2_noise_free_keeps_the_optimum():
    """S:537 example: noise-free scene → both solves reach the known optimum
    (f = 0, GT poses); the dropped 10% do not change the solution."""
    sc = make_scene(10, 300, "unordered", seed=2, vis_prob=0.6)
    first, keep, res, second = xo.xm2(sc)
    assert (~keep).sum() == math.floor(0.1 * sc.E)
    for (dm, st, sol, rep) in (first, second):
        assert st.certified
        assert abs(st.f) <= 1e-8 * (1 + dm.normF)
        assert np.max(np.abs(sol.s - sc.s)) <= 1e-6
        assert np.max(_rot_err(sol.R, sc.R)) <= 1e-6


def test_xm2_removes_outliers():
    """P:569 (greedy outlier removal): with 4% outliers (bearing ±0.3,
    depth ×e^±0.3) the dropped 10% hold most corrupted measurements and the
    second solve's rotations are much closer to the ground truth."""
    from synth.scenes import corrupt
    sc0 = make_scene(12, 400, "unordered", seed=4, vis_prob=0.5, sigma_u=1e-3, sigma_d=0.01)
    sc, bad = corrupt(sc0, 0.04, seed=4)
    first, keep, res, second = xo.xm2(sc)
    assert keep[bad].mean() < 0.2                    # ≥ 80% of the outliers dropped
    assert keep[np.setdiff1d(np.arange(sc.E), bad)].mean() > 0.9
    e1 = np.max(_rot_err(first[2].R, sc.R))
    e2 = np.max(_rot_err(second[2].R, sc.R))
    assert e2 < 0.5 * e1


# ----------------------------------------------------------------------------- tCG (O5)
# Steihaug–Toint truncated CG ("Riemannian trust-region with truncated
# conjugate gradient").  Pins independent of the
# oracle's recurrences: (i) with an unbounded radius and a tiny tolerance the
# returned η solves the projected Newton system H η = −g on the tangent space,
# compared with a dense solve in an explicit orthonormal tangent basis;
# (ii) the scalar recurrences e_Pe, e_Pd, d_Pd equal ⟨η,η⟩, ⟨η,δ⟩, ⟨δ,δ⟩
# recomputed directly; (iii) a boundary / negative-curvature stop puts η on
# the sphere ‖η‖ = Δ; (iv) Hη equals the operator applied to η (linearity).

def _tangent_basis(Y):
    """Orthonormal basis of the tangent space at Y: eigenvectors of the
    (dense) projector matrix with eigenvalue 1."""
    nr = Y.size
    P = np.empty((nr, nr))
    for j in range(nr):
        e = np.zeros(nr)
        e[j] = 1.0
        P[:, j] = xo.project(Y, e.reshape(Y.shape)).ravel()
    P = 0.5 * (P + P.T)
    w, U = np.linalg.eigh(P)
    return U[:, w > 0.5]


def _spd_tangent_operator(Y, seed, cond=50.0, shift=0.0):
    """V ↦ P(A P(V)) for a random symmetric A with spectrum in [1, cond] − shift."""
    rng = np.random.default_rng(seed)
    nr = Y.size
    Qm, _ = np.linalg.qr(rng.standard_normal((nr, nr)))
    A = (Qm * (np.geomspace(1.0, cond, nr) - shift)) @ Qm.T
    A = 0.5 * (A + A.T)

    def hvp(V):
        return xo.project(Y, (A @ xo.project(Y, V).ravel()).reshape(Y.shape))
    return hvp, A


@pytest.mark.parametrize("r", [3, 4])
def test_tcg_unbounded_solves_projected_newton_system(r):
    """Δ = ∞, κ → 0: η = −(TᵀAT)⁻¹Tᵀg expressed in the tangent basis T."""
    Y = random_factor(7, r, 21)
    g = xo.project(Y, random_tangent_ambient(7, r, 22))
    hvp, A = _spd_tangent_operator(Y, 5)
    T = _tangent_basis(Y)
    eta_star = -(T @ np.linalg.solve(T.T @ A @ T, T.T @ g.ravel())).reshape(Y.shape)
    eta, Heta, nh, stop = xo.tcg(hvp, Y, g, 1e12, kappa=1e-13, theta=1.0, max_inner=10 * Y.size)
    assert stop == "converged"
    assert np.linalg.norm(eta - eta_star) <= 1e-9 * np.linalg.norm(eta_star)
    np.testing.assert_allclose(Heta, hvp(eta), atol=1e-9 * np.linalg.norm(Heta))
    # the Newton residual itself (no reference to the recurrences)
    assert np.linalg.norm(hvp(eta) + g) <= 1e-10 * np.linalg.norm(g)


def test_tcg_recurrences_equal_direct_inner_products(small_problem):
    """e_Pe = ⟨η,η⟩, e_Pd = ⟨η,δ⟩, d_Pd = ⟨δ,δ⟩ along the iteration (the boundary
    test ‖η + αδ‖² ≥ Δ² relies on them; Manopt's tCG form)."""
    sc, dm = small_problem
    Y = random_factor(sc.N, 3, 31)
    cases = []
    hvp, _ = _spd_tangent_operator(Y, 6, cond=30.0)
    cases.append((hvp, xo.project(Y, random_tangent_ambient(sc.N, 3, 32))))
    QY = dm.Q @ Y
    g, Lam = xo.rgrad(Y, QY)
    cases.append((lambda V: xo.hess(dm.Q, Y, Lam, V), g))
    for hvp, gg in cases:
        tr = []
        xo.tcg(hvp, Y, gg, 1e12, kappa=1e-10, max_inner=40, trace=tr)
        assert len(tr) >= 3
        g0 = np.linalg.norm(gg)
        for st in tr:
            # absolute scale: ‖η‖·‖δ₀‖ (δ₀ = −g); late δ are at roundoff level
            e, d = st["eta"], st["delta"]
            sc_ = np.linalg.norm(e) * g0
            assert abs(st["e_Pe"] - np.vdot(e, e)) <= 1e-8 * np.vdot(e, e)
            assert abs(st["e_Pd"] - np.vdot(e, d)) <= 1e-8 * sc_
            assert abs(st["d_Pd"] - np.vdot(d, d)) <= 1e-8 * max(np.vdot(d, d), 1e-6 * g0 * g0)


@pytest.mark.parametrize("kind", ["exceeded", "negcurv"])
def test_tcg_truncated_step_lands_on_the_trust_region_boundary(kind):
    """A boundary or negative-curvature stop returns η with ‖η‖ = Δ exactly
    (the positive root τ of ‖η + τδ‖ = Δ)."""
    Y = random_factor(9, 4, 41)
    g = xo.project(Y, random_tangent_ambient(9, 4, 42))
    if kind == "exceeded":
        hvp, A = _spd_tangent_operator(Y, 7, cond=200.0)
        T = _tangent_basis(Y)
        full = np.linalg.norm(T @ np.linalg.solve(T.T @ A @ T, T.T @ g.ravel()))
        Delta = 0.6 * full                         # inside the unbounded solution's norm
    else:
        hvp, A = _spd_tangent_operator(Y, 8, cond=10.0, shift=5.0)   # indefinite
        Delta = 1e6
    eta, Heta, nh, stop = xo.tcg(hvp, Y, g, Delta, kappa=1e-12, max_inner=500)
    assert stop == kind
    assert abs(np.linalg.norm(eta) - Delta) <= 1e-12 * Delta
    np.testing.assert_allclose(Heta, hvp(eta), atol=1e-9 * np.linalg.norm(Heta))
    if kind == "exceeded":
        assert nh >= 2                              # crossed after some CG steps
    # the model decreases along the returned step (Steihaug: m(η) < m(0))
    assert np.vdot(g, eta) + 0.5 * np.vdot(eta, hvp(eta)) < 0.0


def test_tcg_negative_curvature_first_step_is_steepest_descent_to_boundary():
    """H = −I on the tangent space: the first curvature is negative, so η = −Δ g/‖g‖."""
    Y = random_factor(5, 3, 51)
    g = xo.project(Y, random_tangent_ambient(5, 3, 52))
    eta, Heta, nh, stop = xo.tcg(lambda V: -V, Y, g, 0.37)
    assert stop == "negcurv" and nh == 1
    np.testing.assert_allclose(eta, -0.37 * g / np.linalg.norm(g), rtol=0, atol=1e-14)


# ----------------------------------------------------------------------------- App. D (NEXT-3)
# Scale regularisation λ Σ_{i≥2}(X_{3i,3i} − 1)² (App. D);
# on the feasible set X_ii = α_i I₃, so on the factor F = λ Σ_{i≥1}(α_i − 1)².

def _collapse_scene():
    """A noisy forward trajectory whose unregularised optimum collapses the
    scales (F14; App. D's motivation, "collapse all cameras ... into a
    single point"); weights × 1e-3 put ‖Q‖_F ≈ 39 on the scale of λ."""
    sc = make_scene(30, 400, "road", seed=1, sigma_d=0.3, sigma_u=0.05, track_mean=4.0)
    return sc, sc.w * 1e-3


def test_scale_reg_zero_is_the_plain_problem():
    """λ = 0 → the plain solve, bit for bit."""
    sc = make_scene(10, 300, "unordered", seed=3, vis_prob=0.6, sigma_d=0.05, sigma_u=1e-3)
    dm, st, sol, rep = xo.solve(sc)
    dm2, st2, sol2, rep2 = xo.solve(sc, xo.Options(scale_reg=0.0))
    assert np.array_equal(st.Y, st2.Y) and st.f == st2.f and rep["eta"] == rep2["eta"]


@pytest.mark.parametrize("r", [3, 4])
def test_scale_reg_gradient_and_hessian_finite_differences(small_problem, r):
    """d/dh f_λ(R(hV)) = ⟨grad f_λ, V⟩; Euclidean FD of F alone; Hess f_λ[V] =
    P(D grad f_λ[V]); self-adjoint (λ = 2.5 on a random feasible point)."""
    sc, dm = small_problem
    lam = 2.5
    Y = random_factor(sc.N, r, 80 + r)
    V = xo.project(Y, random_tangent_ambient(sc.N, r, 90 + r))
    W = xo.project(Y, random_tangent_ambient(sc.N, r, 95 + r))
    g, Lam = xo.rgrad(Y, dm.Q @ Y, lam)
    h = 1e-5
    fd = (xo.cost(dm.Q, xo.retract(Y, h * V), lam) - xo.cost(dm.Q, xo.retract(Y, -h * V), lam)) / (2 * h)
    assert abs(fd - np.vdot(g, V)) <= 1e-6 * max(1.0, abs(fd))
    # F alone, ambient: ∇F = 2 d_i Y_i (d_0 = 0) — brute force from the definition
    A = random_tangent_ambient(sc.N, r, 99 + r)
    F = lambda Z: lam * sum((np.sum(Z[3 * i:3 * i + 3] ** 2) / 3.0 - 1.0) ** 2 for i in range(1, sc.N))
    fdF = (F(Y + h * A) - F(Y - h * A)) / (2 * h)
    gF = (2.0 * xo.reg_d(Y, lam)[:, None, None] * xo.blocks(Y)).reshape(Y.shape)
    assert abs(fdF - np.vdot(gF, A)) <= 1e-7 * max(1.0, abs(fdF))
    HV = xo.hess(dm.Q, Y, Lam, V, lam)
    h = 1e-6
    gp, _ = xo.rgrad(Y + h * V, dm.Q @ (Y + h * V), lam)
    gm, _ = xo.rgrad(Y - h * V, dm.Q @ (Y - h * V), lam)
    fdH = xo.project(Y, (gp - gm) / (2 * h))
    assert np.linalg.norm(fdH - HV) <= 1e-5 * np.linalg.norm(HV)
    HW = xo.hess(dm.Q, Y, Lam, W, lam)
    assert abs(np.vdot(HV, W) - np.vdot(V, HW)) <= 1e-10 * np.linalg.norm(HV) * np.linalg.norm(W)


def test_scale_reg_prevents_scale_collapse():
    """the unregularised optimum collapses the scales (min s < 0.1); the
    regularised one (λ = 10 ≈ 0.26‖Q‖_F) keeps them (min s ≥ 0.5), certified
    with η ≤ 1e-6."""
    sc, w = _collapse_scene()
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, w)
    st0 = xo.staircase(dm, xo.Options())
    sol0 = xo.round_recover(dm, st0.Y)
    assert st0.certified and sol0.s.min() < 0.1
    st = xo.staircase(dm, xo.Options(scale_reg=10.0))
    sol = xo.round_recover(dm, st.Y, 10.0)
    rep = xo.report(st.cert, sol.rho_hat, dm.normF)
    assert st.certified and sol.s.min() >= 0.5
    assert rep["eta"] <= 1e-6
    # the regulariser only adds a nonnegative term: f_λ ≥ f_0 at the λ-optimum
    assert st.f >= xo.cost(dm.Q, st.Y) - 1e-12 * dm.normF


def test_scale_reg_unit_scale_scene_keeps_the_optimum():
    """noise-free scene with ground-truth scales all 1 ⇒ F vanishes at
    the optimum, λ = 1 gives the same X as λ = 0 (f* = 0, η ≤ 1e-6)."""
    sc = make_scene(12, 300, "unordered", seed=5, vis_prob=0.5, log_scale_range=0.0)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    st0 = xo.staircase(dm, xo.Options())
    st1 = xo.staircase(dm, xo.Options(scale_reg=1.0))
    sol1 = xo.round_recover(dm, st1.Y, 1.0)
    rep1 = xo.report(st1.cert, sol1.rho_hat, dm.normF)
    assert st1.certified and abs(st1.f) <= 1e-8 * dm.normF and rep1["eta"] <= 1e-6
    X0, X1 = st0.Y @ st0.Y.T, st1.Y @ st1.Y.T
    assert np.linalg.norm(X1 - X0) <= 1e-6 * np.linalg.norm(X0)
    np.testing.assert_allclose(sol1.s, 1.0, atol=1e-6)


def test_scale_reg_dual_value_and_Z_by_convexity_identity():
    """App. E proof with F quadratic: for every feasible X′ and the
    certificate (Z_λ, ρ_dual) at x,  f_λ(X′) − ⟨Z_λ, X′⟩ − ρ_dual = F(X′) − F(x) −
    ⟨∇F(x), X′ − x⟩ = λ Σ_{i≥1} (α′_i − α_i)²  (exact Bregman divergence), and
    = ⟨Z_λ, X⟩-gap 0 at x itself when x is critical (strong duality)."""
    sc, w = _collapse_scene()
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, w)
    lam = 10.0
    st = xo.staircase(dm, xo.Options(scale_reg=lam))
    cert = st.cert
    Z = xo.z_matrix(dm.Q, cert.Lam) + np.diag(np.repeat(xo.reg_d(st.Y, lam), 3))
    a = xo.alphas(st.Y)
    for k in range(6):
        Yp = random_factor(sc.N, st.r, 200 + k) if k else st.Y
        ap = xo.alphas(Yp)
        gap = xo.cost(dm.Q, Yp, lam) - np.vdot(Yp, Z @ Yp) - cert.rho_dual
        breg = lam * float(np.sum((ap[1:] - a[1:]) ** 2))
        assert abs(gap - breg) <= 1e-9 * (abs(xo.cost(dm.Q, Yp, lam)) + 1.0), (k, gap, breg)


def test_xm2_select_keeps_every_frame_determined_and_minimal():
    """Readings C22b: after the drop, a frame keeps ≥ 3 measurements of
    landmarks with ≥ 2 kept measurements (pose + scale determined by ≥ 3
    shared points), got back smallest residual first; restored measurements
    whose landmark ends with one kept measurement are dropped again (they add
    nothing to Q, F10 — S:518 minimality)."""
    sc = make_scene(12, 300, "unordered", seed=8, vis_prob=0.5)
    fr, lm = sc.frame.astype(np.int64), sc.landmark.astype(np.int64)
    E = len(fr)
    rng = np.random.default_rng(0)
    res = rng.uniform(0.0, 1.0, E)
    victim = 5
    mine = np.nonzero(fr == victim)[0]
    res[mine] = 10.0 + rng.uniform(0.0, 1.0, mine.size)      # all of frame 5 ranks worst
    # add private (single-view) landmarks of the victim with the worst residuals of all
    extra = 4
    fr = np.concatenate([fr, np.full(extra, victim)])
    lm = np.concatenate([lm, sc.M + np.arange(extra)])
    res = np.concatenate([res, 100.0 + np.arange(extra)])
    M = sc.M + extra
    keep = xo.xm2_select(sc.N, M, fr, lm, res, 0.1)
    kcnt = np.bincount(lm[keep], minlength=M)
    for i in range(sc.N):
        useful = np.sum(keep & (fr == i) & (kcnt[lm] >= 2))
        assert useful >= 3, (i, useful)
    # the victim got back exactly its 3 smallest-residual shared measurements
    back = mine[keep[mine]]
    assert back.size == 3
    assert set(back) == set(mine[np.argsort(res[mine])[:3]])
    # no kept measurement of a private landmark (each would be a single-view leaf)
    assert not keep[E:].any()
    assert xo.connected_components(sc.N, M, fr[keep], lm[keep]) == 1


# ----------------------------------------------------------------------------- NEXT-1
@pytest.mark.parametrize("cfg", [dict(N=10, M=300, kind="unordered", vis_prob=0.6),
                                 dict(N=37, M=900, kind="loop", window=6, sigma_d=0.02,
                                      weights="uniform")], ids=["unordered10", "loop37"])
def test_implicit_Q_apply_equals_the_schur_complement(cfg):
    """NEXT-1: Q·V by the per-edge eliminations of App. A equals the
    dense Schur complement (pinned by brute-force least squares in
    test_prop1_equivalence_brute_force) for r = 1, 3, 5; and ⟨V, QV⟩ = the
    brute-force min_{t,p} Eq. (3) at fixed V (envelope theorem)."""
    sc = make_scene(seed=4, **cfg)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    iq = xo.ImplicitQ(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    for r in (1, 3, 5):
        V = random_tangent_ambient(sc.N, r, 60 + r)
        ref = dm.Q @ V
        assert np.linalg.norm(iq @ V - ref) <= 1e-12 * np.linalg.norm(dm.Q) * np.linalg.norm(V)
    V = random_factor(sc.N, 3, 61)
    assert abs(np.vdot(V, iq @ V) - brute_marginal_objective(sc, V)) <= 1e-8 * (
        1.0 + abs(brute_marginal_objective(sc, V)))


def test_hutchinson_norm_is_unbiased_and_shared():
    """Reading C24: the implicit mode's tolerance scale.  E‖Qz‖² = ‖Q‖_F² for
    Rademacher z: the 16-probe estimate is within its standard error of the
    exact norm, and the implicit and dense products give the same estimate."""
    sc = make_scene(12, 300, "unordered", seed=2, vis_prob=0.5)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    iq = xo.ImplicitQ(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    est_d = xo.hutchinson_normF(lambda Z: dm.Q @ Z, dm.n)
    est_i = xo.hutchinson_normF(iq.apply, dm.n)
    assert abs(est_d - est_i) <= 1e-12 * est_d
    # Var‖Qz‖² = 2(‖Q‖_F⁴ − Σ Q_ii⁴)·… ≤ 2‖Q‖_F⁴: 16 probes ⇒ rel. std of ‖·‖² ≤ √(2/16)
    assert abs(est_d ** 2 - dm.normF ** 2) <= 3 * math.sqrt(2 / 16) * dm.normF ** 2
    many = xo.hutchinson_normF(lambda Z: dm.Q @ Z, dm.n, probes=400)
    assert abs(many ** 2 - dm.normF ** 2) <= 3 * math.sqrt(2 / 400) * dm.normF ** 2


def test_implicit_staircase_reaches_the_dense_optimum():
    """The staircase on the matrix-free operator certifies the same X as on the
    dense Q with the same tolerance scale."""
    sc = make_scene(10, 400, "unordered", seed=6, vis_prob=0.6, sigma_d=0.05, sigma_u=1e-3)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    iq = xo.ImplicitQ(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    nq = xo.hutchinson_normF(iq.apply, dm.n)
    st_i = xo.staircase(iq, normQ=nq)
    st_d = xo.staircase(dm, normQ=nq)
    assert st_i.certified and st_d.certified
    Xi, Xd = st_i.Y @ st_i.Y.T, st_d.Y @ st_d.Y.T
    assert np.linalg.norm(Xi - Xd) <= 1e-6 * np.linalg.norm(Xd)
    assert abs(st_i.f - st_d.f) <= 1e-8 * (1.0 + abs(st_d.f))
