"""Seeded synthetic view graphs shaped like the paper's workloads.

This module is INPUT PLUMBING shared by the oracle (``oracle/``) and the CUDA
path (``paper_2502_04640_b200``).  It holds none of XM's arithmetic: it only
draws ground-truth scenes and produces the lifted 3-D keypoints that the
method consumes (Eq. (2): ũ_ik = d_ik [u_ik; 1]), in the
camera-to-world convention of Eq. (3) (footnote):

    p_k = R_i (s_i ũ_ik) + t_i     ⇔     ũ_ik = s_i⁻¹ R_iᵀ (p_k − t_i)

Frame 0 is the anchored frame (R=I, t=0, s=1).

Scene recipes (restated in DESIGN.md §"Input recipe"):

* ``unordered``  cameras on a sphere (radius 10) looking at the origin,
  landmarks uniform in a ball of radius 2 (depths ≈ 8..12).  Visibility is
  either i.i.d. per (frame, landmark) pair (config A) or per-landmark tracks of
  random length with uniform (config E) or Zipf (config D) frame popularity.
* ``loop``       (Replica-shaped, config B) a camera loop through a 6×6×3 m room
  looking outward; each landmark is a wall point seen by a window of
  consecutive frames ⇒ banded, cyclic co-visibility.
* ``road``       (BAL-Ladybug-shaped, config C) a forward-moving vehicle; each
  landmark is seen by a short run of consecutive frames (banded, open chain).

Noise (applied to the lifted keypoint, not to the GT):
  keypoint σ_u (normalised image units) on u = ũ_xy/ũ_z,
  log-depth Gaussian σ_d: d ← d·exp(σ_d·g),
  App. G model: d ← d·(1+ε)^x, x ~ U(−1, 1).

Every generated graph is connected, has no duplicate (frame, landmark) pair,
every landmark has ≥ 2 observations and every frame ≥ 1.  Same seed ⇒ the
same arrays byte for byte.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass
class Scene:
    N: int
    M: int
    frame: np.ndarray      # int32 [E]
    landmark: np.ndarray   # int32 [E]
    pts: np.ndarray        # float64 [E, 3]  lifted keypoints ũ
    w: np.ndarray          # float64 [E]     weights
    R: np.ndarray          # float64 [N, 3, 3] GT rotations (camera→world)
    t: np.ndarray          # float64 [N, 3]
    s: np.ndarray          # float64 [N]
    p: np.ndarray          # float64 [M, 3]
    name: str = ""
    noise_free: bool = True

    @property
    def E(self) -> int:
        return int(self.frame.shape[0])

    def nbytes_edges(self) -> int:
        return self.E * (4 + 4 + 24 + 8)


# ----------------------------------------------------------------------------
# small geometry helpers (scene construction only)
# ----------------------------------------------------------------------------

def _rand_rot(rng: np.random.Generator, n: int) -> np.ndarray:
    """n uniformly random rotations via unit quaternions."""
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - z * w)
    R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w)
    R[:, 2, 1] = 2 * (y * z + x * w)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _look_at(pos: np.ndarray, target: np.ndarray, up: np.ndarray,
             roll: Optional[np.ndarray] = None) -> np.ndarray:
    """Camera→world rotations whose z axis points from pos to target."""
    z = target - pos
    z /= np.linalg.norm(z, axis=1, keepdims=True)
    x = np.cross(up, z)
    bad = np.linalg.norm(x, axis=1) < 1e-6
    if np.any(bad):
        x[bad] = np.cross(np.array([1.0, 0.0, 0.0]), z[bad])
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y = np.cross(z, x)
    R = np.stack([x, y, z], axis=2)  # columns = camera axes in world
    if roll is not None:
        c, s = np.cos(roll), np.sin(roll)
        Rz = np.zeros((len(roll), 3, 3))
        Rz[:, 0, 0] = c
        Rz[:, 0, 1] = -s
        Rz[:, 1, 0] = s
        Rz[:, 1, 1] = c
        Rz[:, 2, 2] = 1.0
        R = R @ Rz
    return R


def _anchor(R, t, s, p):
    """Re-express the scene so that frame 0 is R=I, t=0, s=1."""
    R0, t0, s0 = R[0].copy(), t[0].copy(), s[0]
    Rn = np.einsum("ji,njk->nik", R0, R)            # R0ᵀ R_i
    tn = (t - t0) @ R0 / s0                           # R0ᵀ (t_i - t0)/s0
    pn = (p - t0) @ R0 / s0
    sn = s / s0
    Rn[0] = np.eye(3)
    tn[0] = 0.0
    sn[0] = 1.0
    return Rn, tn, sn, pn


def _lift(R, t, s, p, frame, landmark):
    """ũ_e = s_i⁻¹ R_iᵀ (p_k − t_i): exact GT keypoints (camera frame)."""
    d = p[landmark] - t[frame]
    u = np.einsum("eji,ej->ei", R[frame], d)
    return u / s[frame][:, None]


def _dedupe_sort(frame, landmark):
    key = frame.astype(np.int64) * (int(landmark.max()) + 1) + landmark
    _, idx = np.unique(key, return_index=True)
    idx.sort()
    return frame[idx], landmark[idx]


def _components(N, M, frame, landmark):
    """Connected components of the bipartite frame–landmark graph (union-find)."""
    parent = np.arange(N + M)

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    # vectorised label propagation is plenty for scene construction
    lab = np.arange(N + M)
    a = frame.astype(np.int64)
    b = N + landmark.astype(np.int64)
    while True:
        m = np.minimum(lab[a], lab[b])
        new = lab.copy()
        np.minimum.at(new, a, m)
        np.minimum.at(new, b, m)
        new = new[new]  # pointer jumping
        if np.array_equal(new, lab):
            break
        lab = new
    del parent, find
    return lab


def _make_connected(N, M, frame, landmark, rng):
    """Append observations until every frame/landmark is present and the
    bipartite graph is connected (scene construction; deterministic in rng)."""
    frame = list(frame)
    landmark = list(landmark)
    fr = np.asarray(frame, dtype=np.int64)
    lm = np.asarray(landmark, dtype=np.int64)
    # every landmark ≥ 2 observations
    cnt = np.bincount(lm, minlength=M)
    for k in np.nonzero(cnt < 2)[0]:
        have = set(fr[lm == k].tolist())
        while len(have) < 2:
            i = int(rng.integers(N))
            if i not in have:
                have.add(i)
                frame.append(i)
                landmark.append(int(k))
    fr = np.asarray(frame, dtype=np.int64)
    lm = np.asarray(landmark, dtype=np.int64)
    # every frame ≥ 1 observation
    fcnt = np.bincount(fr, minlength=N)
    for i in np.nonzero(fcnt == 0)[0]:
        k = int(rng.integers(M))
        frame.append(int(i))
        landmark.append(k)
    fr = np.asarray(frame, dtype=np.int64)
    lm = np.asarray(landmark, dtype=np.int64)
    # connect components by linking a frame of each stray component to a
    # landmark of component 0
    while True:
        lab = _components(N, M, fr, lm)
        roots = np.unique(lab)
        if len(roots) == 1:
            break
        main = lab[0]
        main_lms = np.nonzero(lab[N:] == main)[0]
        for r in roots:
            if r == main:
                continue
            fs = np.nonzero(lab[:N] == r)[0]
            i = int(fs[0])
            k = int(main_lms[rng.integers(len(main_lms))])
            frame.append(i)
            landmark.append(k)
        fr = np.asarray(frame, dtype=np.int64)
        lm = np.asarray(landmark, dtype=np.int64)
    return fr, lm


def _noisy(pts, rng, sigma_u=0.0, sigma_d=0.0, eps=0.0):
    if sigma_u == 0.0 and sigma_d == 0.0 and eps == 0.0:
        return pts.copy()
    d = pts[:, 2].copy()
    u = pts[:, :2] / d[:, None]
    if sigma_u > 0:
        u = u + sigma_u * rng.standard_normal(u.shape)
    if sigma_d > 0:
        d = d * np.exp(sigma_d * rng.standard_normal(d.shape))
    if eps > 0:
        x = rng.uniform(-1.0, 1.0, d.shape)
        d = d * (1.0 + eps) ** x
    out = np.empty_like(pts)
    out[:, :2] = u * d[:, None]
    out[:, 2] = d
    return out


# ----------------------------------------------------------------------------
# scene families
# ----------------------------------------------------------------------------

def _unordered(N, M, rng, vis_prob=None, track_mean=None, track_cap=None,
               zipf=None):
    dirs = rng.standard_normal((N, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    pos = 10.0 * dirs
    R = _look_at(pos, np.zeros((N, 3)) + 0.3 * rng.standard_normal((N, 3)),
                 np.array([0.0, 0.0, 1.0]), roll=rng.uniform(-np.pi, np.pi, N))
    p = rng.standard_normal((M, 3))
    p *= (2.0 * rng.uniform(0, 1, M) ** (1 / 3) / np.linalg.norm(p, axis=1))[:, None]
    if vis_prob is not None:
        mask = rng.uniform(size=(N, M)) < vis_prob
        fr, lm = np.nonzero(mask)
    else:
        # per-landmark tracks: length ~ 2 + Poisson(track_mean - 2), capped
        L = 2 + rng.poisson(max(track_mean - 2.0, 0.0), M)
        L = np.minimum(L, min(track_cap or N, N))
        if zipf is not None:
            pop = 1.0 / np.arange(1, N + 1) ** zipf
            pop = pop[rng.permutation(N)]
        else:
            pop = np.full(N, 1.0)
        pop /= pop.sum()
        cdf = np.cumsum(pop)
        total = int(L.sum())
        # oversample with replacement, dedupe per landmark, top up
        fr_l, lm_l = [], []
        draws = np.searchsorted(cdf, rng.uniform(size=int(total * 1.3) + 16))
        draws = np.minimum(draws, N - 1)
        pos_d = 0
        for k in range(M):
            need = int(L[k])
            chosen = []
            seen = set()
            while len(chosen) < need:
                if pos_d >= len(draws):
                    draws = np.minimum(np.searchsorted(cdf, rng.uniform(size=total + 16)), N - 1)
                    pos_d = 0
                i = int(draws[pos_d])
                pos_d += 1
                if i not in seen:
                    seen.add(i)
                    chosen.append(i)
            fr_l.append(np.asarray(chosen, dtype=np.int64))
            lm_l.append(np.full(need, k, dtype=np.int64))
        fr = np.concatenate(fr_l)
        lm = np.concatenate(lm_l)
    t = pos
    return R, t, p, fr, lm


def _unordered_fast(N, M, rng, track_mean, track_cap, zipf=None):
    """Vectorised per-landmark tracks for large configs (D, E)."""
    dirs = rng.standard_normal((N, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    pos = 10.0 * dirs
    R = _look_at(pos, 0.3 * rng.standard_normal((N, 3)),
                 np.array([0.0, 0.0, 1.0]), roll=rng.uniform(-np.pi, np.pi, N))
    p = rng.standard_normal((M, 3))
    p *= (2.0 * rng.uniform(0, 1, M) ** (1 / 3) / np.linalg.norm(p, axis=1))[:, None]
    L = 2 + rng.poisson(max(track_mean - 2.0, 0.0), M)
    L = np.minimum(L, min(track_cap, N))
    if zipf is not None:
        pop = 1.0 / np.arange(1, N + 1) ** zipf
        pop = pop[rng.permutation(N)]
    else:
        pop = np.full(N, 1.0)
    pop /= pop.sum()
    cdf = np.cumsum(pop)
    fr = np.empty(0, dtype=np.int64)
    lm = np.empty(0, dtype=np.int64)
    need = L.copy()
    rounds = 0
    while need.sum() > 0 and rounds < 64:
        rounds += 1
        ks = np.repeat(np.arange(M), need)
        fs = np.minimum(np.searchsorted(cdf, rng.uniform(size=len(ks))), N - 1)
        fr = np.concatenate([fr, fs])
        lm = np.concatenate([lm, ks])
        key = lm * N + fr
        _, idx = np.unique(key, return_index=True)
        idx.sort()
        fr, lm = fr[idx], lm[idx]
        have = np.bincount(lm, minlength=M)
        need = np.maximum(L - have, 0)
    return R, pos, p, fr, lm


def _loop(N, M, rng, window=12):
    """Replica-shaped: camera loop in a 6×6×3 m room, outward-looking."""
    ang = 2 * np.pi * np.arange(N) / N
    rad = 1.5 + 0.2 * np.sin(3 * ang)
    pos = np.stack([rad * np.cos(ang), rad * np.sin(ang),
                    1.5 + 0.1 * np.sin(5 * ang)], axis=1)
    yaw = ang + 0.25 * np.sin(2 * ang)
    look = pos + np.stack([np.cos(yaw), np.sin(yaw),
                           0.05 * np.sin(7 * ang)], axis=1)
    R = _look_at(pos, look, np.array([0.0, 0.0, 1.0]))
    # landmarks: rays from a start frame hitting the room box [-3,3]²×[0,3]
    i0 = rng.integers(0, N, M)
    Lk = np.clip(rng.poisson(window - 2, M) + 2, 2, 3 * window)
    dirc = np.stack([rng.uniform(-0.5, 0.5, M), rng.uniform(-0.4, 0.4, M),
                     np.ones(M)], axis=1)
    dirc /= np.linalg.norm(dirc, axis=1, keepdims=True)
    dw = np.einsum("mij,mj->mi", R[i0], dirc)
    o = pos[i0]
    tmax = np.full(M, np.inf)
    for ax, lo, hi in ((0, -3.0, 3.0), (1, -3.0, 3.0), (2, 0.0, 3.0)):
        with np.errstate(divide="ignore", invalid="ignore"):
            tl = np.where(dw[:, ax] < 0, (lo - o[:, ax]) / dw[:, ax], np.inf)
            th = np.where(dw[:, ax] > 0, (hi - o[:, ax]) / dw[:, ax], np.inf)
        tmax = np.minimum(tmax, np.minimum(tl, th))
    p = o + tmax[:, None] * dw
    # track = Lk consecutive frames (cyclic) centred on i0
    offs = np.concatenate([np.arange(L) - L // 2 for L in Lk])
    lm = np.repeat(np.arange(M), Lk)
    fr = (np.repeat(i0, Lk) + offs) % N
    return R, pos, p, fr.astype(np.int64), lm.astype(np.int64)


def _road(N, M, rng, track_mean=7.4):
    """BAL-Ladybug-shaped: forward-moving vehicle, landmarks ahead."""
    step = 0.5
    x = step * np.arange(N)
    y = 20.0 * np.sin(x / 150.0)
    z = np.full(N, 1.6)
    pos = np.stack([x, y, z], axis=1)
    dx = np.gradient(x)
    dy = np.gradient(y)
    fwd = np.stack([dx, dy, np.zeros(N)], axis=1)
    R = _look_at(pos, pos + fwd, np.array([0.0, 0.0, 1.0]))
    i0 = rng.integers(0, N, M)
    Lk = np.clip(rng.poisson(track_mean - 2, M) + 2, 2, 24)
    # point ahead of i0 by 14..40 m, lateral ±12, height 0..6 (camera frame)
    qc = np.stack([rng.uniform(-12, 12, M), rng.uniform(-4.4, 1.6, M),
                   rng.uniform(14, 40, M)], axis=1)
    p = pos[i0] + np.einsum("mij,mj->mi", R[i0], qc)
    offs = np.concatenate([np.arange(L) for L in Lk])
    lm = np.repeat(np.arange(M), Lk)
    fr = np.repeat(i0, Lk) + offs
    keep = fr < N
    return R, pos, p, fr[keep].astype(np.int64), lm[keep].astype(np.int64)


# ----------------------------------------------------------------------------
# public entry points
# ----------------------------------------------------------------------------

def make_scene(N: int, M: int, kind: str = "unordered", seed: int = 0, *,
               vis_prob: Optional[float] = None, track_mean: float = 8.0,
               track_cap: int = 1000, zipf: Optional[float] = None,
               window: int = 12, sigma_u: float = 0.0, sigma_d: float = 0.0,
               eps: float = 0.0, weights: str = "unit",
               log_scale_range: float = 0.5, name: str = "") -> Scene:
    """Draw a connected synthetic SBA view graph with known ground truth.

    Parameters mirror SURVEY.md §8(d).  ``weights``: "unit" (w=1) or
    "uniform" (w ~ U(0.5, 1)).  GT scales s_i = exp(U(−a, a)), a =
    ``log_scale_range``; frame 0 anchored.
    """
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), N, M, 0x584D]))
    if kind == "unordered":
        if vis_prob is not None or M * N <= 2_000_000:
            R, t, p, fr, lm = _unordered(N, M, rng, vis_prob=vis_prob,
                                         track_mean=track_mean,
                                         track_cap=track_cap, zipf=zipf)
        else:
            R, t, p, fr, lm = _unordered_fast(N, M, rng, track_mean, track_cap, zipf)
    elif kind == "loop":
        R, t, p, fr, lm = _loop(N, M, rng, window=window)
    elif kind == "road":
        R, t, p, fr, lm = _road(N, M, rng, track_mean=track_mean)
    else:
        raise ValueError(f"unknown scene kind {kind!r}")
    if N > 1:
        fr, lm = _make_connected(N, M, fr, lm, rng)
    else:
        fr = np.zeros(M, dtype=np.int64)
        lm = np.arange(M, dtype=np.int64)
    fr, lm = _dedupe_sort(fr, lm)
    s = np.exp(rng.uniform(-log_scale_range, log_scale_range, N))
    R, t, s, p = _anchor(R, t, s, p)
    pts = _lift(R, t, s, p, fr, lm)
    # drop observations behind / too close to the camera, keep connectivity
    bad = pts[:, 2] < 0.1
    if np.any(bad):
        fr, lm, pts = fr[~bad], lm[~bad], pts[~bad]
        fr2, lm2 = _make_connected(N, M, fr, lm, rng) if N > 1 else (fr, lm)
        if len(fr2) != len(fr):
            fr, lm = _dedupe_sort(fr2, lm2)
            pts = _lift(R, t, s, p, fr, lm)
        if np.any(pts[:, 2] < 0.1):  # last resort: reflect offending depths' landmarks
            raise RuntimeError("scene generation produced non-positive depths")
    noise_free = (sigma_u == 0.0 and sigma_d == 0.0 and eps == 0.0)
    pts = _noisy(pts, rng, sigma_u, sigma_d, eps)
    if weights == "unit":
        w = np.ones(len(fr))
    elif weights == "uniform":
        w = rng.uniform(0.5, 1.0, len(fr))
    else:
        raise ValueError(weights)
    return Scene(N=N, M=M, frame=fr.astype(np.int32), landmark=lm.astype(np.int32),
                 pts=np.ascontiguousarray(pts, dtype=np.float64),
                 w=np.ascontiguousarray(w, dtype=np.float64),
                 R=R, t=t, s=s, p=p, name=name or f"{kind}-N{N}-M{M}-s{seed}",
                 noise_free=noise_free)


#: The five BASELINE.json configurations.
CONFIGS = {
    "A": dict(N=10, M=500, kind="unordered", vis_prob=0.6),
    "B": dict(N=2000, M=100_000, kind="loop", window=12),
    "C": dict(N=1934, M=67_594, kind="road", track_mean=7.4,
              sigma_u=1e-3, sigma_d=0.01),
    "D": dict(N=3765, M=314_000, kind="unordered", track_mean=8.0,
              track_cap=1000, zipf=0.8, sigma_u=1e-3, sigma_d=0.05),
    "E": dict(N=10155, M=33_782, kind="unordered", track_mean=148.0,
              track_cap=2000),
}

CONFIG_DESCRIPTIONS = {
    "A": "synthetic noise-free SBA, N=10 cameras, M=500 points, ~3000 edges",
    "B": "synthetic Replica-shaped sequential trajectory, N=2000 cameras, ~100k points, banded co-visibility, fp64",
    "C": "synthetic BAL Ladybug-shaped, N=1934 cameras, ~0.5M edges, Gaussian keypoint and depth noise",
    "D": "synthetic IMC-shaped unordered scene, N=3765 cameras, irregular co-visibility graph",
    "E": "synthetic BAL Final-shaped, N=10155 cameras, ~5M edges",
}


def config_scene(cfg: str, seed: int = 0, **overrides) -> Scene:
    kw = dict(CONFIGS[cfg])
    kw.update(overrides)
    return make_scene(seed=seed, name=f"cfg{cfg}-s{seed}", **kw)


def random_factor(N: int, r: int, seed: int, anchor_identity: bool = False) -> np.ndarray:
    """Random feasible BM factor Y (n×r): block i = s_i·(r×3 Stiefel)ᵀ.

    Used as a shared random initialisation (Theorem 3 experiments) and as
    random test points.  Returns row-major [3N, r] float64.
    """
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), N, r, 0x5946]))
    Y = np.empty((3 * N, r))
    for i in range(N):
        A = rng.standard_normal((r, 3))
        q, rr = np.linalg.qr(A)
        q = q * np.sign(np.diag(rr))[None, :]
        s = 1.0 if i == 0 else float(np.exp(rng.uniform(-0.5, 0.5)))
        Y[3 * i:3 * i + 3, :] = s * q.T
    if anchor_identity:
        Y[0:3, :] = 0.0
        Y[0:3, 0:3] = np.eye(3)
    return Y


def random_tangent_ambient(N: int, r: int, seed: int) -> np.ndarray:
    """Gaussian ambient matrix n×r (to be projected by the caller)."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), N, r, 0x5456]))
    return rng.standard_normal((3 * N, r))


def splitmix64_uniform(seed: int, n: int) -> np.ndarray:
    """Counter-based uniform(−1,1) stream: x_j = f(splitmix64(seed + j)).

    The same generator is implemented in the CUDA library (Lanczos start
    vector), so both sides can draw the identical vector.  Bits→double:
    (z >> 11) · 2⁻⁵³ ∈ [0,1), then 2u − 1.
    """
    M64 = (1 << 64) - 1
    out = np.empty(n)
    for j in range(n):
        z = (seed + (j + 1) * 0x9E3779B97F4A7C15) & M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        z = z ^ (z >> 31)
        out[j] = 2.0 * ((z >> 11) * (1.0 / 9007199254740992.0)) - 1.0
    return out


def corrupt(sc: Scene, frac: float, seed: int = 0, bearing: float = 0.3, log_depth: float = 0.3):
    """Outlier measurements for XM² tests: a seeded fraction of the
    lifted keypoints gets its normalized image coordinates shifted by
    U(−bearing, bearing) and its depth scaled by exp(U(−log_depth, log_depth))
    (gross but not scale-collapsing; larger corruptions drive the SDP optimum
    to collapsed scales).  Returns (new Scene, sorted indices of
    the corrupted measurements)."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), sc.E, 0x4F55]))
    m = int(round(frac * sc.E))
    idx = np.sort(rng.choice(sc.E, size=m, replace=False))
    pts = sc.pts.copy()
    d = pts[idx, 2].copy()
    u = pts[idx, :2] / d[:, None] + rng.uniform(-bearing, bearing, (m, 2))
    d = d * np.exp(rng.uniform(-log_depth, log_depth, m))
    pts[idx, :2] = u * d[:, None]
    pts[idx, 2] = d
    return dataclasses.replace(sc, pts=pts, noise_free=False, name=sc.name + f"-out{frac:g}"), idx
