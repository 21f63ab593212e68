"""GPU (libxm, sm_100a) vs CPU oracle parity, through the C ABI.

Tolerances (BASELINE.json north_star; readings C12–C15 in DESIGN.md):
  * S co-visibility pattern: bit-exact;
  * Q values: ‖ΔQ‖_F ≤ 1e-10 ‖Q‖_F (κ(K̄)-limited assembly, C13);
  * single SpMM / gradient / HVP on an IDENTICAL Q (oracle Q uploaded with
    xm_set_Q): ‖Δ‖_F ≤ 1e-12 ‖ref‖_F;
  * projection / retraction: ≤ 1e-12 relative;
  * end-to-end: |f_g − f_o| ≤ 1e-8 (1 + |f_o|) (C14), X = YYᵀ ≤ 1e-6 relative
    Frobenius (C12), same certification verdict.
"""
import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import make_scene, random_factor, random_tangent_ambient

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def x_rel_err(Yg, Yo):
    """Exact ‖Y_gY_gᵀ − Y_oY_oᵀ‖_F / ‖Y_oY_oᵀ‖_F via n×n tiles (reading C12)."""
    Xo = Yo @ Yo.T
    return float(np.linalg.norm(Yg @ Yg.T - Xo) / np.linalg.norm(Xo))


SCENES = [
    dict(N=10, M=500, kind="unordered", vis_prob=0.6),                        # config A
    dict(N=37, M=900, kind="loop", window=6),                                # banded, ragged
    dict(N=70, M=1500, kind="road", track_mean=6.0, sigma_u=1e-3, sigma_d=0.01, weights="uniform"),
    dict(N=130, M=2500, kind="unordered", track_mean=10.0, zipf=0.8, sigma_d=0.05, sigma_u=1e-3),
]


@pytest.mark.parametrize("cfg", SCENES, ids=lambda c: f"{c['kind']}{c['N']}")
def test_pattern_bit_exact_and_Q_values(xm, cfg):
    sc = make_scene(seed=3, **cfg)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    with xm.Context() as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        rowptr, colidx = ctx.S_pattern()
        ro, co = xo.s_pattern(sc.N, dm.frame, dm.landmark)
        np.testing.assert_array_equal(rowptr, ro)
        np.testing.assert_array_equal(colidx, co)
        Qg = ctx.Q_rows(0, 3 * sc.N)
    assert np.array_equal(Qg, Qg.T)                       # exactly symmetric
    assert rel(Qg, dm.Q) <= 1e-10, rel(Qg, dm.Q)


def test_duplicates_keep_first_and_errors(xm):
    sc = make_scene(8, 200, "unordered", seed=1, vis_prob=0.5)
    fr = np.concatenate([sc.frame, sc.frame[:5]])
    lm = np.concatenate([sc.landmark, sc.landmark[:5]])
    pts = np.concatenate([sc.pts, sc.pts[:5] * 3.0])       # duplicates carry different data
    w = np.concatenate([sc.w, sc.w[:5]])
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    with xm.Context() as ctx:
        ctx.build_Q(sc.N, sc.M, fr, lm, pts, w)
        assert ctx.stats()["n_dup"] == 5
        assert rel(ctx.Q_rows(0, 3 * sc.N), dm.Q) <= 1e-10
        bad = sc.frame.copy()
        bad[3] = sc.N
        with pytest.raises(xm.XMError) as e:
            ctx.build_Q(sc.N, sc.M, bad, sc.landmark, sc.pts, sc.w)
        assert e.value.name == "EINVAL"
        neg = sc.pts.copy()
        neg[0, 2] = -1.0
        with pytest.raises(xm.XMError):
            ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, neg, sc.w)
    with xm.Context() as ctx:
        with pytest.raises(xm.XMError) as e:
            ctx.build_Q(2, 2, np.array([0, 1]), np.array([0, 1]), np.array([[0.1, 0.1, 1.0]] * 2), None)
        assert e.value.name == "EDISCONNECTED"
        with pytest.raises(xm.XMError) as e:
            ctx.solve()
        assert e.value.name == "ESTATE"


KERNELS = {1: "fullrow", 2: "lowertri"}   # xm_options.spmm_kernel (r > 5 ⇒ full-row)


@pytest.fixture(scope="module", params=sorted(KERNELS), ids=lambda k: KERNELS[k])
def identical_Q(xm, request):
    sc = make_scene(67, 1500, "unordered", seed=5, track_mean=9.0, sigma_d=0.1, sigma_u=0.01)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    ctx = xm.Context(spmm_kernel=request.param)
    ctx.set_Q(dm.Q)
    yield sc, dm, ctx
    ctx.close()


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 7, 12])
def test_spmm_identical_Q(identical_Q, r):
    sc, dm, ctx = identical_Q
    V = random_tangent_ambient(sc.N, r, 100 + r)
    out = ctx.spmm(V)
    ref = dm.Q @ V
    assert rel(out, ref) <= 1e-12
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(dm.Q) * np.linalg.norm(V)


@pytest.mark.parametrize("r", [3, 4, 5, 8])
def test_grad_hvp_project_retract_identical_Q(identical_Q, r):
    sc, dm, ctx = identical_Q
    Y = random_factor(sc.N, r, 200 + r)
    V = xo.project(Y, random_tangent_ambient(sc.N, r, 300 + r))
    W = random_tangent_ambient(sc.N, r, 400 + r)
    g, f = ctx.grad(Y)
    g_o, Lam = xo.rgrad(Y, dm.Q @ Y)
    assert rel(g, g_o) <= 1e-12
    assert abs(f - xo.cost(dm.Q, Y)) <= 1e-12 * abs(xo.cost(dm.Q, Y))
    hv = ctx.hvp(Y, V)
    assert rel(hv, xo.hess(dm.Q, Y, Lam, V)) <= 1e-12
    assert rel(ctx.project(Y, W), xo.project(Y, W)) <= 1e-13
    Yr = ctx.retract(Y, 0.3 * V)
    assert rel(Yr, xo.retract(Y, 0.3 * V)) <= 1e-13


def _e2e(xm, sc, Y0=None, ctx_opts=None, **opts):
    dm, st, sol, rep = xo.solve(sc, Y0=Y0, opts=xo.Options(**opts) if opts else None)
    with xm.Context(**opts, **(ctx_opts or {})) as ctx:  # env switches are read here
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        if Y0 is not None:
            ctx.set_factor(Y0)
        status, info = ctx.solve()
        cert = ctx.certify()
        gsol = ctx.round_recover()
        Yg = ctx.get_factor()
    return dm, st, sol, rep, status, info, cert, gsol, Yg


# tCG code paths on one GPU (xm_create reads these switches): the persistent
# full-row kernel (default), the persistent lower-triangle kernel, one fused
# launch per iteration, and three kernels per iteration in CUDA graphs
TCG_PATHS = {"persist": {"XM_NO_SYM_TCG": "1"}, "persist_sym": {"XM_SYM_TCG": "1"},
             "fused": {"XM_NO_PERSIST_TCG": "1"}, "3kernel": {"XM_NO_FUSED_TCG": "1"}}


@pytest.mark.parametrize("path", sorted(TCG_PATHS))
@pytest.mark.parametrize("kernel", [0, 2], ids=["auto", "lowertri"])
@pytest.mark.parametrize("cfg", SCENES[:3], ids=lambda c: f"{c['kind']}{c['N']}")
def test_end_to_end_solve_parity(xm, cfg, kernel, path, monkeypatch):
    for k, v in TCG_PATHS[path].items():
        monkeypatch.setenv(k, v)
    sc = make_scene(seed=3, **cfg)
    dm, st, sol, rep, status, info, cert, gsol, Yg = _e2e(xm, sc, ctx_opts=dict(spmm_kernel=kernel))
    assert status == 0 and info["certified"] == 1 and st.certified
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    assert x_rel_err(Yg, st.Y) <= 1e-6
    nQ = dm.normF
    # converged λ_min (Lanczos on Z, or shift-invert after the Cholesky of Z + εI)
    assert abs(cert["lambda_min"] - st.cert.lambda_min) <= 1e-6 * nQ
    if cert["lower_rigorous"]:  # Cholesky-proven bound: valid and tight
        assert cert["lambda_lower"] <= st.cert.lambda_min + 1e-9 * nQ
        assert cert["lambda_lower"] >= cert["lambda_min"] - 1e-6 * nQ
        assert cert["eta_rigorous"] >= cert["eta"] - 1e-12
    assert abs(cert["rho_hat"] - sol.rho_hat) <= 1e-8 * (1.0 + abs(sol.rho_hat))
    assert abs(cert["rho_dual"] - st.cert.rho_dual) <= 1e-8 * (1.0 + abs(st.cert.rho_dual))
    assert cert["eta"] <= 1e-6
    np.testing.assert_allclose(gsol["s"], sol.s, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(gsol["R"], sol.R, atol=1e-6)
    np.testing.assert_allclose(gsol["t"], sol.t, atol=1e-6 * max(1.0, np.abs(sol.t).max()))
    np.testing.assert_allclose(gsol["p"], sol.p, atol=1e-6 * max(1.0, np.abs(sol.p).max()))
    assert gsol["n_flipped"] == sol.n_flipped
    if sc.noise_free:   # known optimum (F1): recovered poses = ground truth
        np.testing.assert_allclose(gsol["s"], sc.s, atol=1e-7)
        np.testing.assert_allclose(gsol["R"], sc.R, atol=1e-7)


@pytest.mark.parametrize("path", sorted(TCG_PATHS))
def test_random_init_staircase_parity(xm, path, monkeypatch):
    """Thm 2/3: random init at r=3 escalates to r=4 on both sides, same X."""
    for k, v in TCG_PATHS[path].items():
        monkeypatch.setenv(k, v)
    sc = make_scene(10, 500, "unordered", seed=0, vis_prob=0.6)
    Y0 = random_factor(sc.N, 3, 1)
    dm, st, sol, rep, status, info, cert, gsol, Yg = _e2e(xm, sc, Y0=Y0)
    assert st.ranks == [3, 4]
    assert info["r"] == 4 and info["escapes"] == 1 and status == 0
    assert x_rel_err(Yg, st.Y) <= 1e-6
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))


def test_lanczos_min_eig_matches_dense(xm):
    """Certificate λ_min vs dense brute force on a small Z (uncertified point)."""
    sc = make_scene(12, 300, "unordered", seed=9, vis_prob=0.5, sigma_d=0.1)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    Y = random_factor(sc.N, 4, 5)
    _, Lam = xo.rgrad(Y, dm.Q @ Y)
    lam_d, v_d = xo.dense_min_eig(xo.z_matrix(dm.Q, Lam))
    with xm.Context() as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        ctx.set_factor(Y)
        cert = ctx.certify(want_vector=True)
    assert abs(cert["lambda_min"] - lam_d) <= 1e-8 * dm.normF
    assert abs(abs(float(cert["v"] @ v_d)) - 1.0) <= 1e-6


@pytest.mark.parametrize("path", sorted(TCG_PATHS))
@pytest.mark.parametrize("kernel", [1, 2], ids=["fullrow", "lowertri"])
def test_repeated_solves_reuse_graphs_across_rank_climb(xm, kernel, path, monkeypatch):
    """One context, build → solve twice (as bench.py's steps do) where the
    staircase climbs 3 → 4: the tCG graphs captured at r = 3 in the first solve
    are replayed in the second after the r = 4 products ran, and the results
    are bitwise identical (buffers captured by a graph never move)."""
    for k, v in TCG_PATHS[path].items():
        monkeypatch.setenv(k, v)
    sc = make_scene(10, 500, "unordered", seed=0, vis_prob=0.6)
    Y0 = random_factor(sc.N, 3, 1)
    runs = []
    with xm.Context(spmm_kernel=kernel, profile=1) as ctx:
        for _ in range(3):
            ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
            ctx.set_factor(Y0)
            status, info = ctx.solve()
            runs.append((status, info, ctx.get_factor()))
    for status, info, Y in runs:
        assert status == 0 and info["r"] == 4 and info["escapes"] == 1
        assert info["f"] == runs[0][1]["f"] and np.array_equal(Y, runs[0][2])


@pytest.mark.parametrize("path", ["persist", "persist_sym"])
@pytest.mark.parametrize("r0", [4, 5])
def test_higher_rank_start_parity(xm, path, r0, monkeypatch):
    """Random initial factor at r = 4, 5 (Thm 3: any rank ≥ the optimum's
    certifies): the persistent tCG kernels at R = 4, 5 over > 148 frames
    (every CTA busy, ragged camera split) reach the oracle's X and f."""
    for k, v in TCG_PATHS[path].items():
        monkeypatch.setenv(k, v)
    sc = make_scene(160, 3000, "unordered", seed=5, track_mean=8.0, sigma_u=1e-3, sigma_d=0.02)
    Y0 = random_factor(sc.N, r0, 2)
    dm, st, sol, rep, status, info, cert, gsol, Yg = _e2e(xm, sc, Y0=Y0)
    assert st.certified and status == 0 and info["certified"] == 1 and info["r"] == r0
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    assert x_rel_err(Yg, st.Y) <= 1e-6
    assert np.max(np.abs(gsol["s"] - sol.s)) <= 1e-6
