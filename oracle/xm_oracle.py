"""XM oracle — plain, slow, obviously-correct fp64 CPU implementation.

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2502_04640_b200``) never imports it and
shares no code with it; the only common dependency is the seeded input
generator ``synth/`` (which holds none of the method's arithmetic).

Citations: ``P:n`` = reference PAPER.md line n, ``S:n`` = SPEC.md line n.
Readings of garbled / silent passages follow SURVEY.md §8(c) (C1..C21) and are
listed in DESIGN.md §"Readings".

Conventions (DESIGN.md §"Notation"): the BM factor is stored TALL,
Y = Uᵀ ∈ ℝ^{n×r}, n = 3N, row-major; frame i owns rows 3i..3i+2, the block
Y_i = Ū_iᵀ ∈ ℝ^{3×r}.  Frame 0 is the paper's anchored frame 1.
Inner products are Frobenius over the whole n×r array (reading C4).

Every function is pinned by ``tests/test_oracle_*.py`` against the paper /
mathematics (closed forms, brute force, invariants); no function here is
"parity unpinned".
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

EPS = np.finfo(np.float64).eps


class OracleError(RuntimeError):
    """Raised with one of the status names of include/xm.h (e.g. 'EINVAL')."""

    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


# =============================================================================
# H1  Ingest + validate   (C17)
# =============================================================================

def validate(N: int, M: int, frame, landmark, pts, w=None):
    """Validate a view graph and drop duplicate (frame, landmark) pairs.

    * indices in range, w > 0, finite points, depth ũ_z > 0   (C17)
    * duplicates: keep the first occurrence
    * every frame observed; the bipartite frame–landmark graph restricted to
      observed landmarks is connected (Lemma 1 P:1197 needs it)

    Returns (frame, landmark, pts, w, n_duplicates).
    """
    frame = np.asarray(frame, dtype=np.int64)
    landmark = np.asarray(landmark, dtype=np.int64)
    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    E = frame.shape[0]
    w = np.ones(E) if w is None else np.asarray(w, dtype=np.float64)
    if N < 1 or M < 1 or E < 1:
        raise OracleError("EINVAL", "empty view graph")
    if landmark.shape[0] != E or pts.shape[0] != E or w.shape[0] != E:
        raise OracleError("EINVAL", "array length mismatch")
    if frame.min() < 0 or frame.max() >= N or landmark.min() < 0 or landmark.max() >= M:
        raise OracleError("EINVAL", "index out of range")
    if not (np.all(np.isfinite(pts)) and np.all(np.isfinite(w))):
        raise OracleError("EINVAL", "non-finite value")
    if np.any(w <= 0):
        raise OracleError("EINVAL", "non-positive weight")
    if np.any(pts[:, 2] <= 0):
        raise OracleError("EINVAL", "non-positive depth")
    # keep first duplicate, preserve input order otherwise
    seen = {}
    keep = np.zeros(E, dtype=bool)
    for e in range(E):
        key = (int(frame[e]), int(landmark[e]))
        if key not in seen:
            seen[key] = e
            keep[e] = True
    n_dup = int(E - keep.sum())
    frame, landmark, pts, w = frame[keep], landmark[keep], pts[keep], w[keep]
    if np.any(np.bincount(frame, minlength=N) == 0):
        raise OracleError("EDISCONNECTED", "a frame has no observation")
    if connected_components(N, M, frame, landmark) != 1:
        raise OracleError("EDISCONNECTED", "graph numerically disconnected")
    return frame, landmark, pts, w, n_dup


def connected_components(N: int, M: int, frame, landmark) -> int:
    """Number of components of the bipartite graph on frames ∪ observed
    landmarks, by breadth-first search."""
    adj_f = [[] for _ in range(N)]
    adj_l = {}
    for i, k in zip(np.asarray(frame).tolist(), np.asarray(landmark).tolist()):
        adj_f[i].append(k)
        adj_l.setdefault(k, []).append(i)
    seen_f = [False] * N
    seen_l = set()
    comps = 0
    for s0 in range(N):
        if seen_f[s0]:
            continue
        comps += 1
        stack = [("f", s0)]
        seen_f[s0] = True
        while stack:
            kind, v = stack.pop()
            if kind == "f":
                for k in adj_f[v]:
                    if k not in seen_l:
                        seen_l.add(k)
                        stack.append(("l", k))
            else:
                for i in adj_l[v]:
                    if not seen_f[i]:
                        seen_f[i] = True
                        stack.append(("f", i))
    return comps


# =============================================================================
# H3  Co-visibility (BSR) pattern of S
# =============================================================================

def s_pattern(N: int, frame, landmark):
    """Block pattern {(i,j): i = j or ∃k observed by both i and j}.

    Returned as CSR over frames: rowptr int64 [N+1], colidx int32 sorted per
    row.  This is the structural sparsity of S = H_UU after landmark
    elimination (Q itself is block-dense for connected graphs, F1)."""
    rows = [set([i]) for i in range(N)]
    tracks = {}
    for i, k in zip(np.asarray(frame).tolist(), np.asarray(landmark).tolist()):
        tracks.setdefault(k, []).append(i)
    for fs in tracks.values():
        for a in fs:
            rows[a].update(fs)
    rowptr = np.zeros(N + 1, dtype=np.int64)
    cols = []
    for i in range(N):
        c = sorted(rows[i])
        cols.extend(c)
        rowptr[i + 1] = rowptr[i] + len(c)
    return rowptr, np.asarray(cols, dtype=np.int32)


# =============================================================================
# H4/H5  The data matrix Q   (Prop. 1; App. A)
# =============================================================================

@dataclasses.dataclass
class DataMatrix:
    Q: np.ndarray        # n×n, symmetric PSD (Prop. 1)
    S: np.ndarray        # n×n   H_UU after landmark elimination
    C: np.ndarray        # N×n   H_tU
    K: np.ndarray        # N×N   H_tt
    L: np.ndarray        # Cholesky factor of K̄ = K[1:,1:]   ((N−1)×(N−1))
    G: np.ndarray        # L⁻¹ C̄, C̄ = C[1:, :]             ((N−1)×n)
    W: np.ndarray        # per-landmark total weight W_k = Σ_{e∈k} w_e (Q_3 diag)
    frame: np.ndarray
    landmark: np.ndarray
    pts: np.ndarray
    w: np.ndarray
    N: int
    M: int

    @property
    def n(self):
        return 3 * self.N

    @property
    def normF(self):
        return float(np.linalg.norm(self.Q))


def quadratic_form(N: int, M: int, frame, landmark, pts, w):
    """H = Σ_e w_e b_e b_eᵀ over the stacked variables [Y-rows; t; p].

    The SBA objective Eq. (3) with the unknowns stacked as
    Zext = [Y; T; P] ∈ ℝ^{(3N+N+M)×r} (rows: the 3N rows of Y = Uᵀ, then t_iᵀ,
    then p_kᵀ) is Σ_e w_e ‖b_eᵀ Zext‖² = tr(Zextᵀ H Zext), where b_e has ũ_e
    at rows 3i..3i+2, +1 at t_i and −1 at p_k (App. A P:1161-1167 with
    vec(U) read row-wise; reading C1)."""
    E = len(frame)
    n = 3 * N
    rows = np.repeat(np.arange(E), 5)
    cols = np.empty((E, 5), dtype=np.int64)
    vals = np.empty((E, 5))
    for a in range(3):
        cols[:, a] = 3 * frame + a
        vals[:, a] = pts[:, a]
    cols[:, 3] = n + frame
    vals[:, 3] = 1.0
    cols[:, 4] = n + N + landmark
    vals[:, 4] = -1.0
    B = sp.csr_matrix((vals.ravel(), (rows, cols.ravel())), shape=(E, n + N + M))
    H = (B.T @ sp.diags(w) @ B).tocsr()
    return H


def build_Q(N: int, M: int, frame, landmark, pts, w=None, validate_input=True) -> DataMatrix:
    """Q = Schur complement of H onto the U (Y-row) block after deleting t_0.

    Two exact elimination stages (SURVEY §8(c) "plain definitions"):
      1. landmarks: H_pp = Q_3 = diag(W_k) is diagonal, so
         H_z = H_zz − H_zp diag(W)⁻¹ H_pz exactly (z = [Y-rows; t]);
      2. translations, with t_0 = 0 (anchoring P:137, C2): K̄ = K[1:,1:],
         L = chol(K̄), G = L⁻¹C̄, Q = S − GᵀG   (= S − C̄ᵀ K̄⁻¹ C̄).
    Equivalent to App. A's Q := AᵀQ_tpA + V_tpA + AᵀV_tpᵀ + Q_1 with
    the sign of A corrected (reading C1); the SPEC's principal-submatrix
    choice.  Raises EDISCONNECTED if K̄ is not positive definite.
    """
    if validate_input:
        frame, landmark, pts, w, _ = validate(N, M, frame, landmark, pts, w)
    else:
        frame = np.asarray(frame, np.int64)
        landmark = np.asarray(landmark, np.int64)
        pts = np.asarray(pts, np.float64).reshape(-1, 3)
        w = np.ones(len(frame)) if w is None else np.asarray(w, np.float64)
    n = 3 * N
    H = quadratic_form(N, M, frame, landmark, pts, w)
    nz = n + N
    Hzz = H[:nz, :nz]
    Hzp = H[:nz, nz:]
    Hpp = H[nz:, nz:]
    W = np.asarray(Hpp.diagonal()).copy()
    off = Hpp - sp.diags(W)
    assert off.nnz == 0 or np.abs(off.data).max() == 0.0, "H_pp must be diagonal"
    Winv = np.zeros(M)
    obs = W > 0
    Winv[obs] = 1.0 / W[obs]                    # unobserved landmarks: no term
    Hz = (Hzz - Hzp @ sp.diags(Winv) @ Hzp.T).toarray()
    S = Hz[:n, :n].copy()
    C = Hz[n:, :n].copy()
    K = Hz[n:, n:].copy()
    if N == 1:
        L = np.zeros((0, 0))
        G = np.zeros((0, n))
        Q = S.copy()
    else:
        Kb = K[1:, 1:]
        try:
            L = np.linalg.cholesky(Kb)
        except np.linalg.LinAlgError:
            raise OracleError("EDISCONNECTED", "graph numerically disconnected")
        if np.min(np.diag(L)) <= 1e-12 * math.sqrt(max(np.max(np.abs(np.diag(Kb))), 1e-300)):
            raise OracleError("EDISCONNECTED", "graph numerically disconnected")
        G = sla.solve_triangular(L, C[1:, :], lower=True)
        Q = S - G.T @ G
    Q = 0.5 * (Q + Q.T)
    return DataMatrix(Q=Q, S=S, C=C, K=K, L=L, G=G, W=W, frame=frame, landmark=landmark,
                      pts=pts, w=w, N=N, M=M)


def q_rows(N: int, M: int, frame, landmark, pts, w=None, rows=(), info: Optional[dict] = None
           ) -> np.ndarray:
    """Rows I of the same Q as build_Q, without forming any n×n matrix — the
    full-size sampled parity oracle (configs too large for a dense n×n Q).

    Same definition (Schur complement of Eq. (3)'s quadratic form, landmarks
    then translations eliminated, t_0 = 0; App. A, reading C1):
      * landmark elimination (H_pp = diag(W_k)): for a z-block
        Z (z = [Y-rows; t]),  H_z Z = Σ_e w_e b_e (b_eᵀZ − m_k(e)),
        m_k = Σ_{e∈k} w_e b_eᵀZ / W_k  (the weighted landmark mean);
      * S[I,:] = (H_z E_I)[:n]ᵀ,  C̄[:,I] = (H_z E_I)[n+1:]  (H_z symmetric);
      * K̄ = H_z[t₁.., t₁..] = diag(Σ_{e∈i} w_e) − F diag(1/W) Fᵀ,
        F_ik = Σ_{e: i,k} w_e  (the t-block of the same formula);
      * Q[I,:] = S[I,:] − (K̄⁻¹ C̄[:,I])ᵀ C̄,  with C̄ᵀX = (H_z [0; 0; X])[:n].
    Cost O(E·|I|) plus one dense Cholesky of K̄ ((N−1)×(N−1)).
    If `info` is a dict it receives the rounding-error scale of the
    elimination (reading C13): kappa_K (LAPACK dpocon 1-norm estimate of
    κ(K̄)) and S_I_norm = ‖S[I,:]‖_F (the magnitude Q[I,:] cancels from)."""
    frame, landmark, pts, w, _ = validate(N, M, frame, landmark, pts, w)
    n = 3 * N
    rows = np.asarray(rows, dtype=np.int64).ravel()
    W = np.bincount(landmark, weights=w, minlength=M)
    Winv = np.zeros(M)
    Winv[W > 0] = 1.0 / W[W > 0]

    def hz_apply(Z):                      # Z: (n+N)×c  →  H_z Z
        c = Z.shape[1]
        Yb = Z[:n].reshape(N, 3, c)
        be = np.einsum("ea,eac->ec", pts, Yb[frame]) + Z[n + frame]        # b_eᵀZ
        m = np.zeros((M, c))
        np.add.at(m, landmark, w[:, None] * be)
        res = w[:, None] * (be - Winv[landmark, None] * m[landmark])     # w_e(b_eᵀZ − m_k)
        out = np.zeros((n + N, c))
        outY = out[:n].reshape(N, 3, c)
        np.add.at(outY, frame, pts[:, :, None] * res[:, None, :])
        np.add.at(out[n:], frame, res)
        return out

    def hz_cols(Z, chunk=8):
        return np.concatenate([hz_apply(Z[:, j:j + chunk]) for j in range(0, Z.shape[1], chunk)],
                              axis=1) if Z.shape[1] else np.zeros((n + N, 0))

    EI = np.zeros((n + N, rows.size))
    EI[rows, np.arange(rows.size)] = 1.0
    HI = hz_cols(EI)
    S_I = HI[:n].T.copy()                 # S[I, :]
    if info is not None:
        info.update(S_I_norm=float(np.linalg.norm(S_I)), kappa_K=1.0)
    if N == 1:
        return S_I
    F = sp.csr_matrix((w, (frame, landmark)), shape=(N, M))
    K = -(F @ sp.diags(Winv) @ F.T).toarray()
    K[np.arange(N), np.arange(N)] += np.bincount(frame, weights=w, minlength=N)
    Kb = K[1:, 1:]
    try:
        L = np.linalg.cholesky(Kb)
    except np.linalg.LinAlgError:
        raise OracleError("EDISCONNECTED", "graph numerically disconnected")
    if info is not None:
        rcond, _ = sla.lapack.dpocon(L.T, np.abs(Kb).sum(axis=0).max())
        info["kappa_K"] = 1.0 / max(float(rcond), 1e-300)
    X = sla.cho_solve((L, True), HI[n + 1:])          # K̄⁻¹ C̄[:, I]
    Z = np.zeros((n + N, rows.size))
    Z[n + 1:] = X
    CtX = hz_cols(Z)[:n]                               # C̄ᵀ X
    return S_I - CtX.T


# =============================================================================
# NEXT-1: Q·V without forming Q  ("Extending the XM solver to
# support sparse matrix-vector multiplications")
# =============================================================================

class ImplicitQ:
    """Q = S − C̄ᵀK̄⁻¹C̄ applied to V by the two eliminations of App. A
     on V itself, per edge — the envelope theorem on Eq. (3):
    Q·V = ½∇_V min_{t,p} Σ_e w_e‖V_iᵀũ_e + t_i − p_k‖² (t_0 = 0, reading C2):

      z_e = V_iᵀ ũ_e                        (r-vector per measurement)
      m_k = Σ_{e∈k} w_e z_e / W_k           (landmark mean; H_pp = diag(W))
      b_i = Σ_{e∈i} w_e (z_e − m_k)  = (C̄V)_i,   i ≥ 1
      t   = −K̄⁻¹ b,  t_0 = 0                (the optimal translations, Eq. (4))
      p_k = m_k + Σ_{e∈k} w_e t_{i_e} / W_k  (the optimal landmarks, Eq. (4))
      (QV)_i = Σ_{e∈i} w_e ũ_e (z_e + t_i − p_k)ᵀ

    K̄ = H_tt − H_tp diag(1/W) H_pt without the anchor row / column, factored
    once (Cholesky)."""

    def __init__(self, N: int, M: int, frame, landmark, pts, w=None):
        frame, landmark, pts, w, _ = validate(N, M, frame, landmark, pts, w)
        self.N, self.M, self.n = N, M, 3 * N
        self.frame, self.landmark, self.pts, self.w = frame, landmark, pts, w
        self.W = np.bincount(landmark, weights=w, minlength=M)
        self.Winv = np.zeros(M)
        self.Winv[self.W > 0] = 1.0 / self.W[self.W > 0]
        if N > 1:
            F = sp.csr_matrix((w, (frame, landmark)), shape=(N, M))
            K = -(F @ sp.diags(self.Winv) @ F.T).toarray()
            K[np.arange(N), np.arange(N)] += np.bincount(frame, weights=w, minlength=N)
            self.chol = sla.cho_factor(K[1:, 1:], lower=True)

    def _lm_mean(self, x_e):
        m = np.zeros((self.M, x_e.shape[1]))
        np.add.at(m, self.landmark, self.w[:, None] * x_e)
        return m * self.Winv[:, None]

    def apply(self, V):
        V = np.asarray(V, np.float64)
        r = V.shape[1]
        Vb = V.reshape(self.N, 3, r)
        z = np.einsum("ea,ear->er", self.pts, Vb[self.frame])          # z_e = V_iᵀ ũ_e
        m = self._lm_mean(z)
        t = np.zeros((self.N, r))
        if self.N > 1:
            b = np.zeros((self.N, r))
            np.add.at(b, self.frame, self.w[:, None] * (z - m[self.landmark]))
            t[1:] = -sla.cho_solve(self.chol, b[1:])
        p = m + self._lm_mean(t[self.frame])
        res = self.w[:, None] * (z + t[self.frame] - p[self.landmark])  # w_e (z_e + t_i − p_k)
        out = np.zeros((self.N, 3, r))
        np.add.at(out, self.frame, self.pts[:, :, None] * res[:, None, :])
        return out.reshape(self.n, r)

    def __matmul__(self, V):
        return self.apply(V)

    @property
    def shape(self):
        return (self.n, self.n)


def hutchinson_normF(apply, n: int, probes: int = 16, seed: int = 0x48C0) -> float:
    """‖Q‖_F ≈ √((1/k) Σ_j ‖Q z_j‖²), z_j ∈ {±1}ⁿ = sign of the shared
    counter-based stream (synth.scenes.splitmix64_uniform, seed + j), E[‖Qz‖²]
    = ‖Q‖_F²: the tolerance scale of the implicit mode (reading C24), where Q
    is never formed.  Both sides draw the same probes."""
    from synth.scenes import splitmix64_uniform
    Z = np.stack([np.where(splitmix64_uniform(seed + j, n) < 0.0, -1.0, 1.0) for j in range(probes)],
                 axis=1)
    QZ = apply(Z)
    return math.sqrt(float(np.sum(QZ * QZ)) / probes)


def edge_objective(frame, landmark, pts, w, s, R, t, p) -> float:
    """Eq. (3) evaluated directly: Σ_e w_e ‖s_i R_i ũ_e + t_i − p_k‖²."""
    frame = np.asarray(frame, np.int64)
    landmark = np.asarray(landmark, np.int64)
    pts = np.asarray(pts, np.float64).reshape(-1, 3)
    w = np.ones(len(frame)) if w is None else np.asarray(w, np.float64)
    x_e = s[frame, None] * np.einsum("eab,eb->ea", R[frame], pts) + t[frame]
    resid = x_e - p[landmark]
    return float(np.sum(w * np.sum(resid * resid, axis=1)))


# =============================================================================
# Manifold calculus  (Prop. 4/5 P:360-374; C4, C5)
# =============================================================================

def sym(A):
    """sym(A) = (A + Aᵀ)/2 on the trailing 3×3 axes."""
    return 0.5 * (A + np.swapaxes(A, -1, -2))


def sym0(A):
    """sym₀(A) = sym(A) − (tr A / 3) I₃ (traceless symmetric part)."""
    S = sym(A)
    tr = np.trace(S, axis1=-2, axis2=-1)
    return S - (tr / 3.0)[..., None, None] * np.eye(3)


def blocks(Y):
    """View Y (n×r) as N blocks Y_i ∈ ℝ^{3×r}."""
    n, r = Y.shape
    return Y.reshape(n // 3, 3, r)


def alphas(Y):
    """α_i = ‖Y_i‖_F² / 3 = s_i² (Y_iY_iᵀ = α_i I₃ on the manifold)."""
    B = blocks(Y)
    return np.einsum("ijk,ijk->i", B, B) / 3.0


def multipliers(Y, QY):
    """Λ_i: least-squares solution of (QY)_i = Λ_i Y_i over the constraint
    span of block i (Thm 1 Eq. (18); App. A.4).

    Block 0 (six constraints X_00 = I₃):  Λ_0 = sym((QY)_0 Y_0ᵀ)      (Y_0Y_0ᵀ = I)
    Block i ≥ 1 (B¹..B⁵ = traceless symmetric): Λ_i = sym₀((QY)_i Y_iᵀ)/α_i.
    Returns (N, 3, 3)."""
    B = blocks(Y)
    G = blocks(QY)
    GYt = np.einsum("iar,ibr->iab", G, B)
    Lam = sym0(GYt) / alphas(Y)[:, None, None]
    Lam[0] = sym(GYt[0])
    return Lam


def project(Y, V):
    """Orthogonal (Frobenius) projection onto the tangent space at Y (C4):
    P_i(W) = W − sym₀(W Y_iᵀ) Y_i / α_i   (i ≥ 1: scale × Stiefel),
    P_0(W) = W − sym(W Y_0ᵀ) Y_0          (anchor: Stiefel)."""
    B = blocks(Y)
    W = blocks(V)
    WYt = np.einsum("iar,ibr->iab", W, B)
    Lam = sym0(WYt) / alphas(Y)[:, None, None]
    Lam[0] = sym(WYt[0])
    out = W - np.einsum("iab,ibr->iar", Lam, B)
    return out.reshape(V.shape)


def block_apply(Lam, V):
    """blkdiag(Λ) V."""
    return np.einsum("iab,ibr->iar", Lam, blocks(V)).reshape(V.shape)


# Scale regularisation (App. D; reading C23):
# F(X) = λ Σ_{i≥2} (X_{3i,3i} − 1)², and on the feasible set X_ii = α_i I₃, so on
# the BM factor F = λ Σ_{i≥1} (α_i − 1)² (0-based frames, α_i = ‖Y_i‖²/3).
# Its Euclidean gradient is 2 d_i Y_i with d_i = (2λ/3)(α_i − 1) (d_0 = 0), its
# Hessian along V is 2 d_i V_i + (8λ/9)⟨Y_i, V_i⟩ Y_i.

def reg_d(Y, lam):
    """d_i = (2λ/3)(α_i − 1) for i ≥ 1, d_0 = 0."""
    d = (2.0 * lam / 3.0) * (alphas(Y) - 1.0)
    d[0] = 0.0
    return d


def reg_value(Y, lam):
    """λ Σ_{i≥1} (α_i − 1)²  (App. D objective term)."""
    if lam == 0.0:
        return 0.0
    a = alphas(Y)[1:]
    return lam * float(np.sum((a - 1.0) ** 2))


def reg_delta(Y, D, lam):
    """F(Y + D) − F(Y) without cancellation: λ Σ (α'_i − α_i)(α'_i + α_i − 2),
    α'_i − α_i = ⟨D_i, 2Y_i + D_i⟩/3."""
    if lam == 0.0:
        return 0.0
    B, Db = blocks(Y)[1:], blocks(D)[1:]
    da = np.einsum("iar,iar->i", Db, 2.0 * B + Db) / 3.0
    a = alphas(Y)[1:]
    return lam * float(np.sum(da * (2.0 * a + da - 2.0)))


def cost(Q, Y, lam=0.0):
    """f(Y) = tr(Q U Uᵀ)… = tr(Yᵀ Q Y) = ⟨Y, QY⟩ (Eq. (17)/(23) objective),
    plus the App. D term λ Σ_{i≥1} (α_i − 1)² when λ > 0."""
    return float(np.vdot(Y, Q @ Y)) + reg_value(Y, lam)


def rgrad(Y, QY, lam=0.0):
    """Riemannian gradient = P(2QY) = 2(QY − blkdiag(Λ)Y) = 2 Z(y)Y (C5).
    With λ > 0 (App. D) the regulariser's gradient 2 d_i Y_i is radial, hence
    tangent for i ≥ 1 and without effect on Λ (sym₀ of a multiple of I₃):
    grad = 2(QY + dY − ΛY) = 2 Z_λ(y) Y."""
    Lam = multipliers(Y, QY)
    g = 2.0 * (QY - block_apply(Lam, Y))
    if lam != 0.0:
        g = g + 2.0 * (reg_d(Y, lam)[:, None, None] * blocks(Y)).reshape(Y.shape)
    return g, Lam


def hess(Q, Y, Lam, V, lam=0.0):
    """Riemannian Hessian (analytic HVP; reading C5):
    Hess[V] = P(2QV − 2 blkdiag(Λ) V  [+ 2 d V + (8λ/9)⟨Y_i,V_i⟩ Y_i, App. D])."""
    W = 2.0 * (Q @ V) - 2.0 * block_apply(Lam, V)
    if lam != 0.0:
        B, Vb = blocks(Y), blocks(V)
        yv = np.einsum("iar,iar->i", B, Vb)
        yv[0] = 0.0
        W = W + (2.0 * reg_d(Y, lam)[:, None, None] * Vb
                 + (8.0 * lam / 9.0) * yv[:, None, None] * B).reshape(V.shape)
    return project(Y, W)


def _gram_schmidt_rows(Mx):
    """Modified Gram–Schmidt on the 3 rows of each 3×r block (P:522
    "Gram-Schmidt process on every batch of 3×r matrices"); positive diagonal
    by construction.  Zero pivot → ERETRACT (C20)."""
    out = np.empty_like(Mx)
    for i in range(Mx.shape[0]):
        A = Mx[i].copy()
        scale = np.linalg.norm(A)
        for a in range(3):
            v = A[a].copy()
            for b in range(a):
                v -= np.dot(v, out[i, b]) * out[i, b]
            nv = np.linalg.norm(v)
            if not (nv > 1e-14 * scale):
                raise OracleError("ERETRACT", "retraction failure (zero pivot)")
            out[i, a] = v / nv
    return out


def retract(Y, V, c_floor=1e-3):
    """Retraction on (ℝ₊ × St(r,3))^{N−1} × St(r,3) (readings C6, C7).

    Block i ≥ 1, with s = √α_i, R̂ = Y_i/s:
        δ_s = ⟨V_i, R̂⟩/3,  W = V_i − δ_s R̂,
        s′ = max(s + δ_s, c_f s),  R̂′ = GS(R̂ + W/s),  Y_i′ = s′ R̂′.
    Anchor: Y_0′ = GS(Y_0 + V_0)."""
    B = blocks(Y)
    Vb = blocks(V)
    a = alphas(Y)
    s = np.sqrt(a)
    Rh = B / s[:, None, None]
    ds = np.einsum("iar,iar->i", Vb, Rh) / 3.0
    Wt = Vb - ds[:, None, None] * Rh
    s_new = np.maximum(s + ds, c_floor * s)
    Mx = Rh + Wt / s[:, None, None]
    Mx[0] = B[0] + Vb[0]
    s_new[0] = 1.0
    Rn = _gram_schmidt_rows(Mx)
    return (s_new[:, None, None] * Rn).reshape(Y.shape)


# =============================================================================
# O5  truncated CG (Steihaug–Toint)   (C8)
# =============================================================================

def tcg(hvp, Y, g, Delta, kappa=0.1, theta=1.0, max_inner=500, trace=None):
    """Steihaug–Toint tCG in Manopt's form (no preconditioner).

    Returns (eta, Heta, n_hvp, stop) with stop ∈ {'negcurv', 'exceeded',
    'converged', 'maxinner'}.  If `trace` is a list, the state after every
    completed inner iteration (η, δ, and the scalar recurrences e_Pe = ⟨η,η⟩,
    e_Pd = ⟨η,δ⟩, d_Pd = ⟨δ,δ⟩ that the boundary test uses) is appended to it —
    test instrumentation only, no effect on the arithmetic."""
    eta = np.zeros_like(g)
    Heta = np.zeros_like(g)
    r = g.copy()
    z = float(np.vdot(r, r))
    r0 = math.sqrt(z)
    delta = -r
    e_Pe = 0.0
    e_Pd = 0.0
    d_Pd = z
    n_hvp = 0
    stop = "maxinner"
    for _ in range(max_inner):
        Hd = hvp(delta)
        n_hvp += 1
        d_Hd = float(np.vdot(delta, Hd))
        alpha = z / d_Hd if d_Hd != 0.0 else math.inf
        e_Pe_new = e_Pe + 2.0 * alpha * e_Pd + alpha * alpha * d_Pd
        if d_Hd <= 0.0 or e_Pe_new >= Delta * Delta:
            tau = (-e_Pd + math.sqrt(e_Pd * e_Pd + d_Pd * (Delta * Delta - e_Pe))) / d_Pd
            eta = eta + tau * delta
            Heta = Heta + tau * Hd
            stop = "negcurv" if d_Hd <= 0.0 else "exceeded"
            break
        eta = eta + alpha * delta
        Heta = Heta + alpha * Hd
        e_Pe = e_Pe_new
        r = project(Y, r + alpha * Hd)
        z_old = z
        z = float(np.vdot(r, r))
        if math.sqrt(z) <= r0 * min(r0 ** theta, kappa):
            stop = "converged"
            break
        beta = z / z_old
        delta = -r + beta * delta
        e_Pd = beta * (e_Pd + alpha * d_Pd)
        d_Pd = z + beta * beta * d_Pd
        if trace is not None:
            trace.append(dict(eta=eta.copy(), delta=delta.copy(), e_Pe=e_Pe, e_Pd=e_Pd, d_Pd=d_Pd))
    return eta, Heta, n_hvp, stop


@dataclasses.dataclass
class Options:
    """Defaults: SURVEY §8(c) C7, C8, C11, C19."""
    grad_tol: float = 1e-10          # relative to max(1, ‖Q‖_F)
    delta0_coef: float = 0.1         # Δ₀ = 0.1·√(3N)
    delta_max_mult: float = 10.0     # Δ̄ = 10 Δ₀
    rho_prime: float = 0.1
    tcg_kappa: float = 0.1
    tcg_theta: float = 1.0
    tcg_max_inner: int = 500
    max_outer: int = 5000
    scale_floor: float = 1e-3
    refresh_every: int = 50          # fresh QY every 50 accepted steps (C21)
    eig_tol: float = 1e-8
    cert_tol: float = 1e-6
    lanczos_max: int = 3000
    rank_cap: int = 10
    seed: int = 0
    scale_reg: float = 0.0           # λ of App. D, 0 = the plain problem


@dataclasses.dataclass
class RTRResult:
    Y: np.ndarray
    QY: np.ndarray
    f: float
    grad_norm: float
    converged: bool
    outer: int
    n_hvp: int
    n_spmm: int


def rtr(Q, Y0, opts: Options, normQ: Optional[float] = None) -> RTRResult:
    """Riemannian trust region with tCG (Manopt structure; O4).

    TR ratio with the cancellation-free Δf = 2⟨QY, D⟩ + ⟨D, QD⟩, D = Y′ − Y
    (reading C21), plus the App. D term's change (reg_delta) when λ > 0."""
    lam = opts.scale_reg
    n = Q.shape[0]
    N = n // 3
    normQ = float(np.linalg.norm(Q)) if normQ is None else normQ
    tol = opts.grad_tol * max(1.0, normQ)
    Delta_bar = opts.delta_max_mult * opts.delta0_coef * math.sqrt(3 * N)
    Delta = opts.delta0_coef * math.sqrt(3 * N)
    Y = Y0.copy()
    QY = Q @ Y
    n_spmm = 1
    g, Lam = rgrad(Y, QY, lam)
    f = float(np.vdot(Y, QY)) + reg_value(Y, lam)
    n_hvp = 0
    accepts = 0
    converged = False
    it = 0
    for it in range(opts.max_outer + 1):
        gn = float(np.linalg.norm(g))
        if gn <= tol:
            converged = True
            break
        if it == opts.max_outer:
            break

        def hvp(V):
            return hess(Q, Y, Lam, V, lam)

        eta, Heta, nh, stop = tcg(hvp, Y, g, Delta, opts.tcg_kappa, opts.tcg_theta,
                                  opts.tcg_max_inner)
        n_hvp += nh
        n_spmm += nh
        Yn = retract(Y, eta, opts.scale_floor)
        D = Yn - Y
        QD = Q @ D
        n_spmm += 1
        df = 2.0 * float(np.vdot(QY, D)) + float(np.vdot(D, QD)) + reg_delta(Y, D, lam)
        model_dec = -float(np.vdot(g, eta)) - 0.5 * float(np.vdot(eta, Heta))
        reg = max(1.0, abs(f)) * EPS * 1e3
        rho = (-df + reg) / (model_dec + reg)
        if not (rho >= 0.25) or math.isnan(rho):
            Delta = Delta / 4.0
        elif rho > 0.75 and stop in ("negcurv", "exceeded"):
            Delta = min(2.0 * Delta, Delta_bar)
        if rho > opts.rho_prime:
            Y = Yn
            accepts += 1
            if accepts % opts.refresh_every == 0:
                QY = Q @ Y
                n_spmm += 1
            else:
                QY = QY + QD
            f = float(np.vdot(Y, QY)) + reg_value(Y, lam)
            g, Lam = rgrad(Y, QY, lam)
    QY = Q @ Y                      # fresh before any certificate (O4)
    n_spmm += 1
    g, _ = rgrad(Y, QY, lam)
    return RTRResult(Y=Y, QY=QY, f=float(np.vdot(Y, QY)) + reg_value(Y, lam),
                     grad_norm=float(np.linalg.norm(g)),
                     converged=converged, outer=it, n_hvp=n_hvp, n_spmm=n_spmm)


# =============================================================================
# O6  Certificate: Λ, Z = Q − blkdiag(Λ), λ_min(Z)  (Alg. 1 l.9-12 P:396-402;
#     Thm 1; C10, C11, C19)
# =============================================================================

def z_matrix(Q, Lam):
    """Z(y) = Q − Σ y_i A_i = Q − blkdiag(Λ) (Eq. (16))."""
    Z = Q.copy()
    for i in range(Lam.shape[0]):
        Z[3 * i:3 * i + 3, 3 * i:3 * i + 3] -= Lam[i]
    return Z


def dense_min_eig(Z):
    """Brute force λ_min, v of a small symmetric Z (numpy eigh)."""
    ev, V = np.linalg.eigh(Z)
    v = V[:, 0]
    j = int(np.argmax(np.abs(v)))
    if v[j] < 0:
        v = -v
    return float(ev[0]), v


def lanczos_min_eig(apply_Z, n, tol_abs, max_steps=3000, seed=0):
    """Lanczos with full re-orthogonalisation (reading C19) for the
    smallest eigenpair of a symmetric operator.  Start vector: the shared
    counter-based generator (synth.scenes.splitmix64_uniform).

    Stops when |β_k s_k| ≤ tol_abs for the smallest Ritz pair, or on
    breakdown / max_steps.  Returns (λ_min, v, steps, residual)."""
    from synth.scenes import splitmix64_uniform
    q = splitmix64_uniform(seed, n)
    q /= np.linalg.norm(q)
    Vb = [q]
    alphas_l, betas = [], []
    lam, s_vec, res = math.nan, None, math.inf
    k = 0
    for k in range(1, min(max_steps, n) + 1):
        w = apply_Z(Vb[-1])
        a = float(np.dot(Vb[-1], w))
        alphas_l.append(a)
        Vm = np.array(Vb)
        w = w - Vm.T @ (Vm @ w)          # full re-orthogonalisation (two passes)
        w = w - Vm.T @ (Vm @ w)
        b = float(np.linalg.norm(w))
        if k > 1:   # smallest Ritz pair of the tridiagonal T_k (library eigensolver)
            T_ev, T_vec = sla.eigh_tridiagonal(np.array(alphas_l), np.array(betas),
                                               select="i", select_range=(0, 0))
        else:
            T_ev, T_vec = np.array([a]), np.array([[1.0]])
        lam = float(T_ev[0])
        s_vec = T_vec[:, 0]
        res = abs(b * s_vec[-1])
        if res <= tol_abs or b <= 1e-300 or k == n:
            break
        betas.append(b)
        Vb.append(w / b)
    Vm = np.array(Vb[:len(s_vec)])
    v = Vm.T @ s_vec
    v /= np.linalg.norm(v)
    j = int(np.argmax(np.abs(v)))
    if v[j] < 0:
        v = -v
    return lam, v, k, res


@dataclasses.dataclass
class Certificate:
    lambda_min: float
    v: np.ndarray
    rho_dual: float        # b·y = tr Λ_0
    Lam: np.ndarray
    kkt_resid: float       # ‖Z Y‖_F
    grad_norm: float
    lanczos_steps: int
    trace_X: float


def certificate(Q, Y, opts: Options, QY=None, dense: bool = False, normQ=None) -> Certificate:
    """Λ, Z(y) = Q − blkdiag(Λ) and its smallest eigenpair (Alg. 1 l.9-12).
    With λ > 0 (App. D): Z_λ = Q + λ∇F(X) − Σ y_i A_i = Q + blkdiag(d_i I₃) −
    blkdiag(Λ), and the dual value (App. D/E, "Σ y_i b_i + F(X) − ⟨∇F(X), X⟩")
    ρ_dual = tr Λ_0 + λΣ(α_i − 1)² − Σ 3 d_i α_i = tr Λ_0 − λ Σ_{i≥1}(α_i² − 1)."""
    lam_r = opts.scale_reg
    QY = Q @ Y if QY is None else QY
    g, Lam = rgrad(Y, QY, lam_r)
    normQ = float(np.linalg.norm(Q)) if normQ is None else normQ
    d = reg_d(Y, lam_r) if lam_r != 0.0 else None
    ZY = QY - block_apply(Lam, Y)
    if d is not None:
        ZY = ZY + (d[:, None, None] * blocks(Y)).reshape(Y.shape)
    if dense:
        Z = z_matrix(Q, Lam)
        if d is not None:
            Z = Z + np.diag(np.repeat(d, 3))
        lam, v = dense_min_eig(Z)
        steps = 0
    else:
        def apply_Z(x):
            X = x.reshape(-1, 1)
            out = (Q @ X - block_apply(Lam, X)).ravel()
            if d is not None:
                out = out + np.repeat(d, 3) * x
            return out
        lam, v, steps, _ = lanczos_min_eig(apply_Z, Q.shape[0],
                                           opts.eig_tol * max(1.0, normQ),
                                           opts.lanczos_max, opts.seed)
    rho_dual = float(np.trace(Lam[0]))
    if lam_r != 0.0:
        a = alphas(Y)[1:]
        rho_dual -= lam_r * float(np.sum(a * a - 1.0))
    return Certificate(lambda_min=lam, v=v, rho_dual=rho_dual, Lam=Lam,
                       kkt_resid=float(np.linalg.norm(ZY)), grad_norm=float(np.linalg.norm(g)),
                       lanczos_steps=steps, trace_X=float(np.vdot(Y, Y)))


# =============================================================================
# O7  Riemannian staircase (Algorithm 1; Thm 2; C9)
# =============================================================================

def escape(Q, Y, QY, v, max_halvings=60, c_floor=1e-3, lam=0.0):
    """Y₊ = Retr_{[Y,0]}(α[0, v]) with α = 1, ½, … until f decreases
    (Alg. 1 l.14-22; D = [0; vᵀ] is tangent at [Y, 0], Thm 2, reading C9).
    Δf computed cancellation-free (C21).  Returns (Y₊, α, Δf)."""
    n, r = Y.shape
    Yz = np.concatenate([Y, np.zeros((n, 1))], axis=1)
    QYz = np.concatenate([QY, np.zeros((n, 1))], axis=1)
    Dir = np.zeros((n, r + 1))
    Dir[:, r] = v
    alpha = 1.0
    for _ in range(max_halvings + 1):
        Yp = retract(Yz, alpha * Dir, c_floor)
        D = Yp - Yz
        df = 2.0 * float(np.vdot(QYz, D)) + float(np.vdot(D, Q @ D)) + reg_delta(Yz, D, lam)
        if df < 0.0:
            return Yp, alpha, df
        alpha *= 0.5
    raise OracleError("EESCAPE", "escape failed")


@dataclasses.dataclass
class StaircaseResult:
    Y: np.ndarray
    QY: np.ndarray
    f: float
    r: int
    certified: bool
    converged: bool
    cert: Certificate
    ranks: list
    n_hvp: int
    n_spmm: int
    outer: int


def staircase(dm_or_Q, opts: Options = None, Y0=None, r0=3, dense_cert=False,
              normQ: Optional[float] = None) -> StaircaseResult:
    """Algorithm 1: init U⁰ = [I₃,…,I₃] at r = 3 unless Y0 is given.
    `normQ` overrides ‖Q‖_F as the tolerance scale (the implicit mode's
    estimate, reading C24); Q may be an ImplicitQ (matrix-free products)."""
    opts = opts or Options()
    Q = dm_or_Q.Q if isinstance(dm_or_Q, DataMatrix) else dm_or_Q
    n = Q.n if isinstance(Q, ImplicitQ) else Q.shape[0]
    N = n // 3
    normQ = float(np.linalg.norm(Q)) if normQ is None else float(normQ)
    if Y0 is None:
        Y = np.zeros((n, r0))
        for i in range(N):
            Y[3 * i:3 * i + 3, 0:3] = np.eye(3)
    else:
        Y = np.array(Y0, dtype=np.float64)
    ranks = [Y.shape[1]]
    n_hvp = n_spmm = outer = 0
    while True:
        res = rtr(Q, Y, opts, normQ)
        n_hvp += res.n_hvp
        n_spmm += res.n_spmm
        outer += res.outer
        cert = certificate(Q, res.Y, opts, QY=res.QY, dense=dense_cert, normQ=normQ)
        ok = cert.lambda_min >= -opts.cert_tol * max(1.0, normQ)
        r = res.Y.shape[1]
        if ok or not res.converged or r >= opts.rank_cap:
            return StaircaseResult(Y=res.Y, QY=res.QY, f=res.f, r=r,
                                   certified=bool(ok and res.converged),
                                   converged=res.converged, cert=cert, ranks=ranks,
                                   n_hvp=n_hvp, n_spmm=n_spmm, outer=outer)
        Y, _, _ = escape(Q, res.Y, res.QY, cert.v, c_floor=opts.scale_floor, lam=opts.scale_reg)
        ranks.append(Y.shape[1])


# =============================================================================
# O8  Rounding + recovery  (Eq. (4), Eq. (9) P:219-234;
#     S:436-471; C16, C20)
# =============================================================================

def _polar(B):
    U, sv, Vt = np.linalg.svd(B)
    return U @ Vt, U, sv, Vt


@dataclasses.dataclass
class Solution:
    R: np.ndarray       # (N,3,3) SO(3), camera→world (Eq. (3))
    s: np.ndarray       # (N,)
    t: np.ndarray       # (N,3)
    p: np.ndarray       # (M,3)  (NaN for unobserved landmarks)
    n_flipped: int
    Yr: np.ndarray      # rounded, gauge-fixed factor (n×3) = Ūᵀ
    rho_hat: float      # f(Yr) = tr(Q Ū ᵀŪ)
    edge_objective: float  # Eq. (3) evaluated directly at (R, s, t, p)


def round_recover(dm: DataMatrix, Y, lam: float = 0.0) -> Solution:
    """Rounding: top-3 eigenvectors of X = YYᵀ via the r×r Gram YᵀY,
    Y₃ = Y W₃; per block: s_i = ‖B_i‖_F/√3, polar → O(3); gauge fix
    U* = R̄_0ᵀ Ū (Eq. (12)) with s_0 renormalised to 1 (C16);
    det < 0 ⇒ nearest SO(3) (Eq. (9)).  Recovery (Eq. (4)):
    T = −K̄⁻¹ C̄ Y₃ (t_0 = 0), p_k = Σ_{e∈k} w_e (Ū_i ũ_e + t_i)/W_k."""
    N, M = dm.N, dm.M
    n, r = Y.shape
    ev, Wv = np.linalg.eigh(Y.T @ Y)
    W3 = Wv[:, ::-1][:, :3] if r >= 3 else Wv
    Y3 = Y @ W3
    Ub = blocks(Y3).transpose(0, 2, 1)       # Ū_i = Y3_iᵀ (3×3)
    O0, _, _, _ = _polar(Ub[0])
    s0 = np.linalg.norm(Ub[0]) / math.sqrt(3.0)
    if not s0 > 1e-12:
        raise OracleError("EDEGENERATE", "degenerate block")
    Ub = np.einsum("ba,ibc->iac", O0, Ub) / s0     # O0ᵀ Ū_i / s0
    R = np.empty((N, 3, 3))
    s = np.empty(N)
    flips = 0
    for i in range(N):
        si = np.linalg.norm(Ub[i]) / math.sqrt(3.0)
        if not si > 1e-12:
            raise OracleError("EDEGENERATE", "degenerate block")
        Ri, U, sv, Vt = _polar(Ub[i])
        if np.linalg.det(Ri) < 0:
            U = U.copy()
            U[:, 2] = -U[:, 2]
            Ri = U @ Vt
            flips += 1
        R[i], s[i] = Ri, si
    R[0] = np.eye(3)
    s[0] = 1.0
    Ubar = s[:, None, None] * R
    Yr = Ubar.transpose(0, 2, 1).reshape(n, 3)
    # Eq. (4): translations, then landmarks
    t = np.zeros((N, 3))
    if N > 1:
        t[1:] = -sla.cho_solve((dm.L, True), dm.C[1:, :] @ Yr)
    x_e = np.einsum("eab,eb->ea", Ubar[dm.frame], dm.pts) + t[dm.frame]
    p = np.full((M, 3), np.nan)
    acc = np.zeros((M, 3))
    np.add.at(acc, dm.landmark, dm.w[:, None] * x_e)
    obs = dm.W > 0
    p[obs] = acc[obs] / dm.W[obs, None]
    edge_obj = edge_objective(dm.frame, dm.landmark, dm.pts, dm.w, s, R, t, p)
    return Solution(R=R, s=s, t=t, p=p, n_flipped=flips, Yr=Yr,
                    rho_hat=float(np.vdot(Yr, dm.Q @ Yr)) + reg_value(Yr, lam),
                    edge_objective=edge_obj)


# =============================================================================
# O9  Report: suboptimality   (Eq. (13); App. E; C10)
# =============================================================================

def suboptimality(rho_hat, rho_lower):
    """η = (ρ̂ − ρ_lower)/(1 + |ρ̂| + |ρ_lower|)   (Eq. (13))."""
    return (rho_hat - rho_lower) / (1.0 + abs(rho_hat) + abs(rho_lower))


def report(cert: Certificate, rho_hat: float, normQ: float = 1.0, cert_tol: float = 1e-6):
    """η per Eq. (13) with ρ_SDP bounded below as SURVEY §8(c) O9 /
    reading C10 state it:  ρ_lower = ρ_dual + min(0, λ_min)·tr X̂  (ρ_dual =
    b·y = tr Λ_0, strong duality P:340, Thm 1; the min(0, ·) term is the
    correction for a Z(y) that is not exactly PSD — a heuristic when λ_min < 0,
    C10).  η_E per App. E as printed (max(0, λ_min))."""
    rho_lower = cert.rho_dual + min(0.0, cert.lambda_min) * cert.trace_X
    lowE = max(0.0, cert.lambda_min) * cert.trace_X + cert.rho_dual
    return dict(rho_lower=rho_lower, eta=suboptimality(rho_hat, rho_lower),
                eta_E=(rho_hat - lowE) / (1.0 + abs(rho_hat) + abs(lowE)),
                certified=cert.lambda_min >= -cert_tol * max(1.0, normQ))


def solve(scene_or_arrays, opts: Options = None, Y0=None, dense_cert=False):
    """End to end: build Q → staircase → certificate → round/recover → report."""
    s = scene_or_arrays
    dm = build_Q(s.N, s.M, s.frame, s.landmark, s.pts, s.w)
    st = staircase(dm, opts, Y0=Y0, dense_cert=dense_cert)
    sol = round_recover(dm, st.Y, (opts or Options()).scale_reg)
    rep = report(st.cert, sol.rho_hat, dm.normF, (opts or Options()).cert_tol)
    return dm, st, sol, rep


# =============================================================================
# XM² — drop the largest-residual measurements and solve again
# ("delete the 10% measurements with the largest residuals and re-run the
# XM solver … XM² (running twice)"; S:472-476 edge_residuals
# xm_squared; reading C22 in DESIGN.md)
# =============================================================================

def edge_residuals(frame, landmark, pts, w, sol: Solution) -> np.ndarray:
    """The summands of Eq. (3):
    res_e = w_e ‖s_i R_i ũ_e + t_i − p_k‖² at a recovered solution.
    Their sum is `edge_objective`."""
    frame = np.asarray(frame, np.int64)
    landmark = np.asarray(landmark, np.int64)
    pts = np.asarray(pts, np.float64).reshape(-1, 3)
    w = np.ones(len(frame)) if w is None else np.asarray(w, np.float64)
    res = np.empty(len(frame))
    for e in range(len(frame)):                      # one observation at a time
        i, k = frame[e], landmark[e]
        d = sol.s[i] * (sol.R[i] @ pts[e]) + sol.t[i] - sol.p[k]
        res[e] = w[e] * float(d @ d)
    return res


def xm2_select(N: int, M: int, frame, landmark, res, drop_fraction: float = 0.1,
               min_obs: int = 3) -> np.ndarray:
    """Which measurements XM² keeps (readings C22, C22b).

    1. Order the E measurements by residual, largest first; equal residuals
       by (landmark, frame) ascending.  Drop the first ⌊drop_fraction·E⌋.
    2. Keep every frame determined (C22b): a frame needs ≥ min_obs kept
       measurements of landmarks that have ≥ 2 kept measurements (its pose
       and scale then follow from ≥ 3 shared points).  Frames in ascending
       order; a deficient frame gets its dropped measurements back in the
       reverse of the drop order (smallest residual first) until it has
       min_obs such measurements (or none are left).
    3. Never disconnect: if some frame is no longer in the
       component of the others (bipartite frame–landmark graph of the kept
       measurements), restore dropped measurements in the reverse of the drop
       order, each one only if it joins two components, until all frames are
       in one component (S:518's "restore minimal edges by ascending residual
       until connected").
    4. Minimality: a restored measurement whose landmark ends with a
       single kept measurement adds nothing to Q (F10) — dropped again.
    Returns a boolean keep mask over the E measurements."""
    frame = np.asarray(frame, np.int64)
    landmark = np.asarray(landmark, np.int64)
    E = len(frame)
    nd = int(math.floor(drop_fraction * E))
    order = sorted(range(E), key=lambda e: (-res[e], int(landmark[e]), int(frame[e])))
    dropped = order[:nd]
    keep = np.ones(E, dtype=bool)
    keep[dropped] = False
    restored = np.zeros(E, dtype=bool)
    # 2. determined frames
    kcnt = np.bincount(landmark[keep], minlength=M)
    rank = np.empty(E, dtype=np.int64)
    rank[np.asarray(order, dtype=np.int64)] = np.arange(E)
    by_frame = [[] for _ in range(N)]
    for e in range(E):
        by_frame[int(frame[e])].append(e)
    for i in range(N):
        def useful():
            return sum(1 for e in by_frame[i] if keep[e] and kcnt[landmark[e]] >= 2)
        cand = sorted((e for e in by_frame[i] if not keep[e]), key=lambda e: -rank[e])
        for e in cand:
            if useful() >= min_obs:
                break
            keep[e] = True
            restored[e] = True
            kcnt[landmark[e]] += 1
    # 3. connectivity (Kruskal over the remaining dropped list, smallest residual first)
    parent = list(range(N + M))                      # frames 0..N-1, landmarks N..N+M-1

    def find(x):
        while parent[x] != x:
            x = parent[x]
        return x

    for e in np.nonzero(keep)[0]:
        a, b = find(int(frame[e])), find(N + int(landmark[e]))
        if a != b:
            parent[b] = a
    has_frame = {}
    for i in range(N):
        has_frame[find(i)] = True
    n_frame_comps = len(has_frame)
    for e in reversed(dropped):                      # smallest residual first
        if n_frame_comps == 1:
            break
        if keep[e]:
            continue
        a, b = find(int(frame[e])), find(N + int(landmark[e]))
        if a == b:
            continue
        fa, fb = has_frame.get(a, False), has_frame.get(b, False)
        parent[b] = a
        has_frame[a] = fa or fb
        keep[e] = True
        restored[e] = True
        if fa and fb:
            n_frame_comps -= 1
    # 4. minimality: restored leaves (landmark with one kept measurement) go again
    kcnt = np.bincount(landmark[keep], minlength=M)
    leaf = restored & keep & (kcnt[landmark] == 1)
    keep[leaf] = False
    return keep


def xm2(scene, opts: Options = None, drop_fraction: float = 0.1, dense_cert=False):
    """XM²: solve, rank the (de-duplicated) measurements by
    `edge_residuals` at the recovered solution, keep `xm2_select`'s set,
    rebuild Q and solve again.  Returns (first, keep, residuals, second) with
    first / second = solve()'s (dm, staircase, solution, report)."""
    s = scene
    first = solve(s, opts, dense_cert=dense_cert)
    fr, lm, pts, w, _ = validate(s.N, s.M, s.frame, s.landmark, s.pts, s.w)
    res = edge_residuals(fr, lm, pts, w, first[2])
    keep = xm2_select(s.N, s.M, fr, lm, res, drop_fraction)
    s2 = dataclasses.replace(s, frame=fr[keep].astype(np.int32), landmark=lm[keep].astype(np.int32),
                             pts=pts[keep], w=w[keep]) if dataclasses.is_dataclass(s) else \
        type("Scene2", (), dict(N=s.N, M=s.M, frame=fr[keep], landmark=lm[keep], pts=pts[keep], w=w[keep]))
    second = solve(s2, opts, dense_cert=dense_cert)
    return first, keep, res, second
