"""One Steihaug–Toint tCG solve on the
device vs the pinned oracle tCG (tests/test_oracle_pins.py::test_tcg_*), on an
IDENTICAL Q (oracle Q uploaded with xm_set_Q), through the C ABI (xm_tcg):
same stop reason, same HVP count, η and Hη ≤ 1e-10 relative — for every
device implementation of the loop (persistent lower-triangle, persistent
full-row, one fused launch per iteration, three kernels per iteration)."""
import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import make_scene, random_factor, random_tangent_ambient

pytestmark = pytest.mark.gpu

PATHS = ["persist_sym", "persist", "fused", "three_kernel"]


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


SCENES = {
    "loop37": dict(N=37, M=900, kind="loop", window=6),
    "unordered130": dict(N=130, M=2500, kind="unordered", track_mean=10.0, zipf=0.8,
                         sigma_d=0.05, sigma_u=1e-3),
}


def points(sc, dm, r):
    """A random feasible point (indefinite Hessian, large gradient) and a point
    near the oracle's optimum (PSD Hessian, small gradient)."""
    out = [("random", random_factor(sc.N, r, 17))]
    st = xo.staircase(dm, xo.Options(), r0=3)
    Ys = st.Y if st.Y.shape[1] == r else np.concatenate(
        [st.Y, np.zeros((st.Y.shape[0], r - st.Y.shape[1]))], axis=1)
    V = xo.project(Ys, random_tangent_ambient(sc.N, r, 18))
    out.append(("near_opt", xo.retract(Ys, 1e-2 * V / np.linalg.norm(V) * np.sqrt(sc.N))))
    return out


@pytest.mark.parametrize("scene", list(SCENES))
@pytest.mark.parametrize("r", [3, 4])
def test_tcg_matches_oracle_on_every_path(xm, scene, r):
    sc = make_scene(seed=5, **SCENES[scene])
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    ran = set()
    with xm.Context() as ctx:
        ctx.set_Q(dm.Q)
        for label, Y in points(sc, dm, r):
            g, Lam = xo.rgrad(Y, dm.Q @ Y)

            def hvp(V):
                return xo.hess(dm.Q, Y, Lam, V)
            eta_big, _, _, _ = xo.tcg(hvp, Y, g, 1e6)
            for Delta in (1e6, 0.3 * np.linalg.norm(eta_big)):
                eo, Ho, no, so = xo.tcg(hvp, Y, g, Delta)
                for path in PATHS:
                    try:
                        eg, Hg, ng, sg = ctx.tcg(Y, Delta, path)
                    except xm.XMError as e:
                        assert e.code == -1, e          # path not available for (N, r)
                        continue
                    ran.add(path)
                    ctx_msg = (scene, r, label, Delta, path)
                    assert sg == so and ng == no, (ctx_msg, sg, so, ng, no)
                    assert rel(eg, eo) <= 1e-10, (ctx_msg, rel(eg, eo))
                    assert rel(Hg, Ho) <= 1e-10, (ctx_msg, rel(Hg, Ho))
                    if so in ("exceeded", "negcurv"):
                        assert abs(np.linalg.norm(eg) - Delta) <= 1e-12 * Delta
    assert {"persist_sym", "three_kernel"} <= ran, ran
