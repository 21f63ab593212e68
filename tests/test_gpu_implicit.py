"""SURVEY §8(f) NEXT-1 on the device: Q·V without forming Q (P:1075,
xm_options.implicit_q), through the C ABI, against the pinned oracle
(xm_oracle.ImplicitQ / the dense Schur complement, hutchinson_normF;
test_oracle_pins.py::test_implicit_*): single products ≤ 1e-12 relative to
‖Q‖‖V‖ for r = 1..12, the shared 16-probe tolerance scale, and the solve →
certificate → recovery against the oracle's dense solve with the same
tolerance scale (f, X, λ_min, ρ̂, R, s, t)."""
import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import config_scene, make_scene, random_factor, random_tangent_ambient

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


SCENES = [
    dict(N=10, M=500, kind="unordered", vis_prob=0.6),
    dict(N=70, M=1500, kind="road", track_mean=6.0, sigma_u=1e-3, sigma_d=0.01, weights="uniform"),
    dict(N=160, M=3000, kind="unordered", track_mean=10.0, zipf=0.8, sigma_d=0.05, sigma_u=1e-3),
]


@pytest.mark.parametrize("cfg", SCENES, ids=lambda c: f"{c['kind']}{c['N']}")
def test_implicit_products_and_norm(xm, cfg):
    sc = make_scene(seed=3, **cfg)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    iq = xo.ImplicitQ(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    with xm.Context(implicit_q=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        for r in (1, 3, 4, 5, 7, 12):
            V = random_tangent_ambient(sc.N, r, 40 + r)
            out = ctx.spmm(V)
            scale = np.linalg.norm(dm.Q) * np.linalg.norm(V)
            assert np.linalg.norm(out - dm.Q @ V) <= 1e-12 * scale, r
            assert np.linalg.norm(out - iq @ V) <= 1e-12 * scale, r
        status, info = ctx.solve()
    # the tolerance scale: the same 16 Rademacher probes on both sides (C24)
    est = xo.hutchinson_normF(iq.apply, dm.n)
    assert abs(info["normQ"] - est) <= 1e-10 * est


@pytest.mark.parametrize("cfg", SCENES, ids=lambda c: f"{c['kind']}{c['N']}")
def test_implicit_grad_and_hvp(xm, cfg):
    """The Riemannian gradient and HVP (reading C5) through the
    matrix-free products: ≤ 1e-12 relative against the oracle's rgrad / hess
    on the dense Q, at random feasible points, r = 3, 4, 5."""
    sc = make_scene(seed=3, **cfg)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    with xm.Context(implicit_q=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        for r in (3, 4, 5):
            Y = random_factor(sc.N, r, 200 + r)
            V = xo.project(Y, random_tangent_ambient(sc.N, r, 300 + r))
            g, f = ctx.grad(Y)
            g_o, Lam = xo.rgrad(Y, dm.Q @ Y)
            assert np.linalg.norm(g - g_o) <= 1e-12 * np.linalg.norm(g_o), r
            assert abs(f - xo.cost(dm.Q, Y)) <= 1e-12 * abs(xo.cost(dm.Q, Y)), r
            hv = ctx.hvp(Y, V)
            h_o = xo.hess(dm.Q, Y, Lam, V)
            assert np.linalg.norm(hv - h_o) <= 1e-12 * np.linalg.norm(h_o), r


@pytest.mark.parametrize("cfg", SCENES, ids=lambda c: f"{c['kind']}{c['N']}")
def test_implicit_solve_matches_dense_oracle(xm, cfg):
    sc = make_scene(seed=3, **cfg)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    iq = xo.ImplicitQ(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    est = xo.hutchinson_normF(iq.apply, dm.n)
    st = xo.staircase(dm, normQ=est)
    sol = xo.round_recover(dm, st.Y)
    with xm.Context(implicit_q=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
        Yg = ctx.get_factor()
    assert status == 0 and info["certified"] == 1 and st.certified
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    Xo = st.Y @ st.Y.T
    assert np.linalg.norm(Yg @ Yg.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
    assert abs(cert["lambda_min"] - st.cert.lambda_min) <= 1e-6 * est
    assert abs(cert["rho_hat"] - sol.rho_hat) <= 1e-8 * (1.0 + abs(sol.rho_hat))
    assert cert["eta"] <= 1e-6
    np.testing.assert_allclose(g["s"], sol.s, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(g["R"], sol.R, atol=1e-6)
    np.testing.assert_allclose(g["t"], sol.t, atol=1e-6 * max(1.0, np.abs(sol.t).max()))


def test_implicit_E_sampled_products_and_known_optimum(xm):
    """Config E matrix-free: sampled rows of Q·V against oracle.q_rows (the
    reading-C13 tolerance), and the noise-free scene's known optimum."""
    sc = config_scene("E")
    rng = np.random.default_rng(5)
    frames = np.unique(np.concatenate([[0, 1, sc.N - 1], rng.integers(0, sc.N, 8)]))
    rows = np.sort((3 * frames[:, None] + np.arange(3)).ravel())
    info_q = {}
    QI = xo.q_rows(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w, rows, info=info_q)
    V = random_tangent_ambient(sc.N, 3, 9)
    ref = QI @ V
    tol = max(1e-10, 8 * np.finfo(float).eps * info_q["kappa_K"] * info_q["S_I_norm"] / np.linalg.norm(QI))
    with xm.Context(implicit_q=1) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
        out = ctx.spmm(V)
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
    assert np.linalg.norm(out[rows] - ref) <= tol * np.linalg.norm(ref)
    assert status == 0 and info["certified"] == 1
    assert abs(info["f"]) <= 1e-8 * info["normQ"] and cert["eta"] <= 1e-6
    np.testing.assert_allclose(g["s"], sc.s, atol=1e-7)
    np.testing.assert_allclose(g["R"], sc.R, atol=1e-7)


def test_conditional_graph_loop_equals_batched_graphs(xm, monkeypatch):
    """The tCG loop as ONE conditional-WHILE graph launch runs exactly the
    kernels of the batched graphs up to the stop: the same trajectory, bitwise
    (matrix-free products, three-kernel tCG iterations)."""
    sc = make_scene(seed=7, N=300, M=4000, kind="unordered", track_mean=12.0, sigma_d=0.01, sigma_u=1e-3)
    runs = []
    for flag in (None, "1"):
        if flag:
            monkeypatch.setenv("XM_NO_COND_GRAPH", flag)
        else:
            monkeypatch.delenv("XM_NO_COND_GRAPH", raising=False)
        with xm.Context(implicit_q=1) as ctx:
            ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
            status, info = ctx.solve()
            runs.append((status, info, ctx.get_factor()))
    (s0, i0, Y0), (s1, i1, Y1) = runs
    assert s0 == s1 == 0
    assert i0["hvps"] == i1["hvps"] and i0["outer_iters"] == i1["outer_iters"]
    assert i0["f"] == i1["f"] and np.array_equal(Y0, Y1)
