"""many small instances in one launch (xm_solve_batch;
one CTA runs the whole Algorithm 1 per instance), against the pinned oracle's
staircase instance by instance: Thm 3's random-initialisation trials
on one shared Q, and an App. G-style noise sweep with one Q per
instance, in the shared-memory layout (N ≤ 24) and the global-memory layout
(BAL-93's N = 93, the size of the paper's 1000 trials).  Tolerances as the
single-instance end-to-end parity (C12, C14):
f ≤ 1e-8(1 + |f|), X = YYᵀ ≤ 1e-6, same certification, λ_min ≤ 1e-6‖Q‖_F."""
import numpy as np
import pytest

from oracle import xm_oracle as xo
from synth.scenes import make_scene, random_factor

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xm():
    from paper_2502_04640_b200 import xm as _xm
    _xm.load_library()
    return _xm


def identity_start(N, r=3):
    Y = np.zeros((3 * N, r))
    for i in range(N):
        Y[3 * i:3 * i + 3, :3] = np.eye(3)
    return Y


def check_against_oracle(Q, Y0, Yg, res):
    st = xo.staircase(Q, Y0=Y0)
    assert res["certified"] == int(st.certified) == 1, res
    assert res["status"] == 0
    assert abs(res["f"] - st.f) <= 1e-8 * (1.0 + abs(st.f))
    r = res["r"]
    Yd = Yg[:, :r]
    assert np.abs(Yg[:, r:]).max(initial=0.0) == 0.0          # unused columns stay zero
    Xo = st.Y @ st.Y.T
    assert np.linalg.norm(Yd @ Yd.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
    assert abs(res["lambda_min"] - st.cert.lambda_min) <= 1e-6 * max(1.0, np.linalg.norm(Q))
    return st


def test_random_init_trials_reach_the_global_optimum(xm):
    """Thm 3: from random feasible starts the staircase reaches the
    unique optimum of a noise-free scene — every trial, and each of a sample
    equal to the oracle's staircase from the same start."""
    sc = make_scene(10, 500, "unordered", seed=0, vis_prob=0.6)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    B = 64
    Y0 = np.stack([random_factor(sc.N, 3, 1000 + b) for b in range(B)])
    with xm.Context() as ctx:
        Yg, res = ctx.solve_batch(dm.Q, Y0, shared_Q=True)
    Xgt = None
    for b in range(B):
        assert res[b]["certified"] == 1 and res[b]["status"] == 0, (b, res[b])
        Y = Yg[b][:, :res[b]["r"]]
        X = Y @ Y.T
        Xgt = X if Xgt is None else Xgt
        assert np.linalg.norm(X - Xgt) <= 1e-6 * np.linalg.norm(Xgt)      # one optimum
        assert abs(res[b]["f"]) <= 1e-8 * dm.normF
    assert sum(r["r"] > 3 for r in res) >= 1        # some trials needed a staircase escape
    for b in (0, 1, 2, 17, 40, 63):
        check_against_oracle(dm.Q, Y0[b], Yg[b], res[b])


def test_noise_sweep_one_Q_per_instance(xm):
    """App. G-style sweep: the same view graph at increasing depth noise, one Q
    per instance, identity starts (Alg. 1 line 4); every instance vs the oracle."""
    levels = [0.0, 0.01, 0.03, 0.1, 0.2, 0.3]
    Qs, scs = [], []
    for k, sd in enumerate(levels):
        sc = make_scene(16, 300, "unordered", seed=4, vis_prob=0.5, sigma_d=sd, sigma_u=sd / 20)
        scs.append(sc)
        Qs.append(xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w).Q)
    Q = np.stack(Qs)
    Y0 = np.stack([identity_start(16) for _ in levels])
    with xm.Context() as ctx:
        Yg, res = ctx.solve_batch(Q, Y0)
    for b in range(len(levels)):
        check_against_oracle(Q[b], Y0[b], Yg[b], res[b])


def test_batch_matches_the_single_instance_path(xm):
    """The batched kernel and xm_solve (the streaming path) reach the same X."""
    sc = make_scene(20, 600, "loop", seed=2, window=5, sigma_d=0.02, sigma_u=1e-3)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    with xm.Context() as ctx:
        Yg, res = ctx.solve_batch(dm.Q, identity_start(20)[None], shared_Q=True)
        ctx.set_Q(dm.Q)
        st, info = ctx.solve()
        Ys = ctx.get_factor()
    Yb = Yg[0][:, :res[0]["r"]]
    Xs = Ys @ Ys.T
    assert st == 0 and res[0]["certified"] == 1
    assert np.linalg.norm(Yb @ Yb.T - Xs) <= 1e-6 * np.linalg.norm(Xs)


def bal93_scene(seed=0):
    """BAL-93-shaped (Thm 3's "1000 trials" ran on BAL-93): 93 cameras,
    61203 points, mean track 4.7 (≈ 287k observations), small keypoint / depth
    noise — n = 279, past the shared-memory layout (global-memory layout)."""
    return make_scene(93, 61203, "unordered", seed=seed, track_mean=4.7, sigma_u=1e-3, sigma_d=0.01)


def test_large_instances_random_init_trials(xm):
    """Thm 3 at the paper's size (BAL-93): random feasible starts on one shared
    Q (global-memory layout), every trial certified at the same X, and a sample
    equal to the oracle's staircase from the same start."""
    sc = bal93_scene()
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    B = 24
    Y0 = np.stack([random_factor(sc.N, 3, 2000 + b) for b in range(B)])
    with xm.Context() as ctx:
        Yg, res = ctx.solve_batch(dm.Q, Y0, shared_Q=True)
    Xref = None
    for b in range(B):
        assert res[b]["certified"] == 1 and res[b]["status"] == 0, (b, res[b])
        Y = Yg[b][:, :res[b]["r"]]
        X = Y @ Y.T
        Xref = X if Xref is None else Xref
        assert np.linalg.norm(X - Xref) <= 1e-6 * np.linalg.norm(Xref)
    for b in (0, 7, 23):
        check_against_oracle(dm.Q, Y0[b], Yg[b], res[b])


def test_large_instance_matches_the_single_instance_path(xm):
    """Global-memory layout vs xm_solve (streaming path) from the identity start."""
    sc = make_scene(40, 2000, "unordered", seed=5, track_mean=6.0, sigma_u=1e-3, sigma_d=0.01)
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    with xm.Context() as ctx:
        Yg, res = ctx.solve_batch(dm.Q, identity_start(40)[None], shared_Q=True)
        ctx.set_Q(dm.Q)
        st, info = ctx.solve()
        Ys = ctx.get_factor()
    Yb = Yg[0][:, :res[0]["r"]]
    Xs = Ys @ Ys.T
    assert st == 0 and res[0]["certified"] == 1
    assert np.linalg.norm(Yb @ Yb.T - Xs) <= 1e-6 * np.linalg.norm(Xs)
    check_against_oracle(dm.Q, identity_start(40), Yg[0], res[0])


def test_batch_rejects_oversized_instances(xm):
    with xm.Context() as ctx:
        with pytest.raises(xm.XMError) as e:
            ctx.solve_batch(np.zeros((1203, 1203)), identity_start(401)[None], shared_Q=True)
    assert e.value.code == -1
