"""SURVEY §8(f) NEXT-3 on the device: the scale-regularised objective of
App. D, f_λ = ⟨Y, QY⟩ + λ Σ_{i≥1}(α_i − 1)², its modified
Z_λ = Q + blkdiag(2λ/3 (α_i − 1) I) − blkdiag(Λ) and dual value
tr Λ_0 − λΣ(α_i² − 1), against the pinned oracle (test_oracle_pins.py
::test_scale_reg_*), through the C ABI (xm_options.scale_reg)."""
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


def collapse_scene():
    sc = make_scene(30, 400, "road", seed=1, sigma_d=0.3, sigma_u=0.05, track_mean=4.0)
    return sc, sc.w * 1e-3


@pytest.mark.parametrize("r", [3, 4])
def test_gradient_and_hvp_identical_Q(xm, r):
    sc = make_scene(37, 900, "loop", seed=2, window=6, sigma_d=0.02, sigma_u=1e-3)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    lam = 3.7
    Y = random_factor(sc.N, r, 12)
    V = xo.project(Y, random_tangent_ambient(sc.N, r, 13))
    g_o, Lam = xo.rgrad(Y, dm.Q @ Y, lam)
    H_o = xo.hess(dm.Q, Y, Lam, V, lam)
    f_o = xo.cost(dm.Q, Y, lam)
    with xm.Context(scale_reg=lam) as ctx:
        ctx.set_Q(dm.Q)
        g, f = ctx.grad(Y)
        H = ctx.hvp(Y, V)
    assert rel(g, g_o) <= 1e-12 and abs(f - f_o) <= 1e-12 * abs(f_o)
    assert rel(H, H_o) <= 1e-12


def test_lambda_zero_is_the_plain_solve(xm):
    sc = make_scene(37, 900, "loop", seed=2, window=6, sigma_d=0.02, sigma_u=1e-3)
    out = []
    for opts in ({}, {"scale_reg": 0.0}):
        with xm.Context(**opts) as ctx:
            ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
            status, info = ctx.solve()
            out.append((ctx.get_factor(), info["f"], info["hvps"]))
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1:] == out[1][1:]


def test_collapse_scene_matches_oracle(xm):
    sc, w = collapse_scene()
    lam = 10.0
    dm, st, sol, rep = xo.solve(_with_w(sc, w), xo.Options(scale_reg=lam))
    st0 = xo.staircase(dm, xo.Options())
    with xm.Context(scale_reg=lam) as ctx:
        ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, w)
        status, info = ctx.solve()
        cert = ctx.certify()
        g = ctx.round_recover()
        Yg = ctx.get_factor()
    with xm.Context() as ctx0:
        ctx0.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, w)
        ctx0.solve()
        g0 = ctx0.round_recover()
    assert g0["s"].min() < 0.1                                  # unregularised: collapsed
    assert status == 0 and info["certified"] == 1 and st.certified
    assert g["s"].min() >= 0.5                                  # App. D keeps the scales
    assert abs(info["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    Xo = st.Y @ st.Y.T
    assert np.linalg.norm(Yg @ Yg.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
    assert abs(cert["lambda_min"] - st.cert.lambda_min) <= 1e-6 * dm.normF
    assert abs(cert["rho_dual"] - st.cert.rho_dual) <= 1e-8 * (1.0 + abs(st.cert.rho_dual))
    assert abs(cert["rho_hat"] - sol.rho_hat) <= 1e-8 * (1.0 + abs(sol.rho_hat))
    assert cert["eta"] <= 1e-6 and rep["eta"] <= 1e-6
    np.testing.assert_allclose(g["s"], sol.s, rtol=1e-6)
    np.testing.assert_allclose(g["R"], sol.R, atol=1e-6)


def _with_w(sc, w):
    import dataclasses
    return dataclasses.replace(sc, w=w)
