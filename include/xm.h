/*
 * xm.h — C ABI of libxm, the B200 (sm_100a) hot path of XM
 * ("Building Rome with Convex Optimization", arXiv 2502.04640).
 *
 * Citations: P:n = reference PAPER.md line n, S:n = SPEC.md line n.
 *
 * The library computes, on one or more B200s (one process per GPU):
 *   xm_build_Q        the marginalised data matrix Q of Prop. 1 (P:153-184,
 *                     App. A) from a view graph of depth-lifted
 *                     keypoints (Eq. (2), Eq. (3));
 *   xm_solve          Algorithm 1, the Riemannian staircase with a
 *                     Riemannian trust-region / truncated-CG local solver
 *                      on the BM factorisation (Prop. 4/5,
 *                     P:360-374), certifying each rank with the dual
 *                     matrix Z(y) = Q − Σ y_i A_i (Eq. (16), Thm 1);
 *   xm_certify        the certificate at the final point: λ_min(Z), ρ_dual,
 *                     the rounded objective ρ̂ and η (Eq. (13), App. E);
 *   xm_round_recover  rounding, gauge fixing (Eq. (12)),
 *                     SO(3) projection (Eq. (9)) and recovery of
 *                     translations / landmarks (Eq. (4)).
 *
 * Memory: every array argument may be HOST memory (pageable or pinned) or
 * DEVICE memory on the context's device (e.g. a torch CUDA tensor); the
 * library detects which with cudaPointerGetAttributes and copies as needed.
 * Inputs are caller-owned and only read during the call.  Outputs are written
 * to caller-allocated buffers before the call returns.  The context owns all
 * of its device memory (freed by xm_destroy).
 *
 * Layouts: row-major, 0-based.  Frame 0 is the paper's anchored frame 1
 * (R = I, t = 0, s = 1).  The BM factor is exchanged TALL:
 * Y = Uᵀ ∈ ℝ^{n×r}, n = 3N, frame i owns rows 3i..3i+2 (Y_i = Ū_iᵀ).
 *
 * Errors: every entry point returns an xm_status; nothing throws across the
 * ABI.  A failed call leaves the context in its previous stage (except
 * XM_ECUDA / XM_ENCCL, after which the context must be destroyed).
 *
 * Threading: a context is not thread-safe; independent contexts are
 * independent.  Multi-GPU: one process per GPU; every rank passes the
 * same full inputs and calls every function collectively; outputs are
 * identical on all ranks.
 *
 * Call order: xm_create → xm_build_Q → xm_solve → xm_certify →
 * xm_round_recover (xm_set_Q may replace xm_build_Q for tests).  Calling out
 * of order returns XM_ESTATE.
 */
#ifndef XM_H_
#define XM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  XM_OK = 0,              /* certified (xm_solve) / success                       */
  XM_UNCERTIFIED = 2,     /* converged but λ_min(Z) < −cert_tol at the rank cap    */
  XM_NOT_CONVERGED = 3,   /* trust region hit max_outer before the gradient tol   */
  XM_EINVAL = -1,         /* bad argument: index out of range, w ≤ 0, ũ_z ≤ 0,    */
                          /* non-finite value, r out of range        */
  XM_EDISCONNECTED = -2,  /* "graph numerically disconnected"        */
  XM_ENOMEM = -3,         /* device allocation failed                              */
  XM_ECUDA = -4,          /* CUDA runtime error (context unusable)                 */
  XM_ENCCL = -5,          /* NCCL error (context unusable)                         */
  XM_ERETRACT = -6,       /* "retraction failure": zero Gram–Schmidt pivot */
  XM_EESCAPE = -7,        /* "escape failed": 60 halvings without decrease*/
  XM_EINFEASIBLE = -8,    /* "infeasible point": rank-deficient block     */
  XM_EDEGENERATE = -9,    /* "degenerate block" / scale collapse s_i < 1e-8*/
  XM_ESTATE = -10         /* call order violated                                    */
} xm_status;

typedef struct xm_ctx xm_ctx;

/* Solver options.  Defaults (xm_default_options): SURVEY §8(c) C7, C8, C11,
 * C19 — the paper prints none. */
typedef struct {
  double grad_tol;        /* stop when ‖grad‖ ≤ grad_tol·max(1,‖Q‖_F)   [1e-10] */
  double delta0_coef;     /* initial TR radius Δ₀ = coef·√(3N)              [0.1] */
  double delta_max_mult;  /* Δ̄ = mult·Δ₀                                    [10]  */
  double rho_prime;       /* acceptance threshold ρ′                        [0.1] */
  double tcg_kappa;       /* tCG stop ‖r‖ ≤ r₀·min(r₀^θ, κ)                 [0.1] */
  double tcg_theta;       /*                                                [1.0] */
  double eig_tol;         /* Lanczos residual ≤ eig_tol·max(1,‖Q‖_F)       [1e-8] */
  double cert_tol;        /* certified iff λ_min ≥ −cert_tol·max(1,‖Q‖_F)  [1e-6] */
  double scale_floor;     /* scale retraction s′ = max(s+δ, c·s), c         [1e-3] */
  int32_t tcg_max_inner;  /*                                                [500] */
  int32_t max_outer;      /* per staircase rank                            [5000] */
  int32_t rank_cap;       /* Algorithm 1 stops climbing at this r (≤ 12)    [10]  */
  int32_t lanczos_max;    /* Lanczos step cap                              [3000] */
  int32_t refresh_every;  /* fresh Q·Y every k accepted TR steps (C21)       [50] */
  int32_t profile;        /* 1: time every SpMM with CUDA events (xm_stats)  [0]  */
  int32_t cert_cholesky;  /* 1: if Lanczos has not converged within n/72 steps,  */
                          /* test Z + εI ⪰ 0 by dense Cholesky (ε = cert_tol·   */
                          /* max(1,‖Q‖_F); Alg. 1); single GPU     [1]  */
  int32_t spmm_kernel;    /* Q·V kernel: 0 auto by (N, r); 1 full-row stream;  */
                          /* 2 lower-triangle (symmetric) stream — one GPU and */
                          /* r ≤ 5 only, else falls back to 1 [0] */
  uint64_t seed;          /* Lanczos start vector (splitmix64 stream)         [0]  */
  double scale_reg;       /* λ of the scale-regularised objective of App. D  */
                          /* (P:1612-1655): f + λ Σ_{i≥1} (α_i − 1)², Z_λ =   */
                          /* Q + blkdiag(2λ/3 (α_i−1) I) − blkdiag(Λ), dual   */
                          /* tr Λ_0 − λ Σ (α_i² − 1).  λ > 0 uses the unfused */
                          /* product + epilogue kernels (no persistent tCG)  [0]  */
  int32_t implicit_q;     /* 1: never form Q: each   */
                          /* Q·V by per-measurement elimination passes + K̄⁻¹ */
                          /* (world > 1: pass shares + a K̄⁻¹ band, five       */
                          /* all-reduces); ‖Q‖_F by a 16-probe estimate (C24); */
                          /* certificate by Lanczos on Z only.  0: dense Q.   */
                          /* −1: by a per-product time model at xm_build_Q    */
                          /* (E: matrix-free on 1–2 GPUs; A–D: dense)   [−1]  */
} xm_options;

typedef struct {
  double f;               /* final objective tr(Q UᵀU) = ⟨Y, QY⟩            */
  double grad_norm;       /* final Riemannian gradient norm                   */
  double lambda_min;      /* λ_min(Z) at the final rank                        */
  double normQ;           /* ‖Q‖_F                                             */
  double s_min;           /* min_i s_i at the final point                      */
  int32_t r;              /* final rank                                         */
  int32_t certified;      /* 1 if λ_min ≥ −cert_tol·max(1,‖Q‖_F) and converged */
  int32_t converged;
  int32_t escapes;        /* number of staircase escapes (rank lifts)           */
  int64_t outer_iters;
  int64_t hvps;           /* tCG Hessian-vector products                        */
  int64_t spmms;          /* all Q·V products (HVP, Δf, fresh QY, escapes)      */
  int64_t lanczos_steps;
} xm_solve_info;

typedef struct {
  double lambda_min;      /* λ_min(Z(y)), Z = Q − blkdiag(Λ) (Eq. (16)): converged */
                          /* Lanczos on Z (method 0) or shift-invert Lanczos on  */
                          /* (Z + εI)⁻¹ after its Cholesky (method 1)            */
  double lambda_lower;    /* lower bound on λ_min: if lower_rigorous, proven by a */
                          /* completed Cholesky of Z + δI and its backward error */
                          /* (−δ − γ_{n+1}·tr(Z+δI) − u‖Z‖_F); else = λ_min      */
  double rho_dual;        /* b·y = tr Λ_0 (dual objective, Eq. (16))      */
  double rho_hat;         /* objective at the rounded, recovered solution        */
  double rho_lower;       /* ρ_dual + min(0, λ_min)·tr X̂ (reading C10)          */
  double eta;             /* (ρ̂ − ρ_lower)/(1 + |ρ̂| + |ρ_lower|)  (Eq. (13))    */
  double eta_E;           /* App. E formula as printed: max(0, λ_min)·tr X       */
  double rho_lower_rigorous; /* ρ_dual + min(0, λ_lower)·tr X̂                   */
  double eta_rigorous;    /* Eq. (13) with rho_lower_rigorous                    */
  double kkt_resid;       /* ‖Z(y) Y‖_F (Thm 1 Eq. (18))                         */
  double grad_norm;
  double trace_X;         /* tr X = ‖Y‖_F²                                      */
  double normQ;
  int32_t lanczos_steps;
  int32_t certified;
  int32_t method;         /* 0: Lanczos on Z; 1: Cholesky of Z + εI + shift-invert */
  int32_t lower_rigorous; /* 1: lambda_lower is the Cholesky-proven bound        */
} xm_certificate;

typedef struct {
  int64_t kernel_launches;   /* every kernel launched by this context            */
  int64_t spmm_calls;
  int64_t spmm_rows;         /* Q rows streamed per call on this rank            */
  double spmm_ms;            /* Σ CUDA-event time of SpMM launches (profile=1)  */
  int64_t spmm_timed;        /* number of SpMM launches included in spmm_ms      */
  double spmm_alg_bytes;     /* Σ algorithmic bytes of those launches:           */
                             /*   8·(nrows·n + n·r + nrows·r) each               */
  double ms_build, ms_solve, ms_certify, ms_round;  /* host wall per phase        */
  int64_t n_dup;             /* duplicate observations dropped (keep first)     */
  int64_t E;                 /* observations after de-duplication                */
  int64_t nnzb_S;            /* blocks in S's co-visibility pattern              */
  int64_t q_bytes;           /* bytes of Q streamed by one SpMM on this rank     */
} xm_stats;

/* ------------------------------------------------------------------------ */
void xm_default_options(xm_options* opts);
const char* xm_strerror(xm_status s);

/* Create a context on CUDA `device`.  rank/world: this process's place in the
 * row sharding (world = 1: single GPU).  nccl_id: 128-byte ncclUniqueId from
 * xm_nccl_unique_id on rank 0, broadcast by the caller (NULL if world == 1).
 * opts: NULL ⇒ defaults.  cuda_stream: a cudaStream_t to run on (NULL ⇒ the
 * context creates its own non-blocking stream).
 * Testing world > 1 on one GPU: an nccl_id whose first bytes are
 * XM_LOOPBACK_MAGIC joins an in-process loopback group instead of NCCL — the
 * `world` contexts (one host thread each, same 128-byte id) then exchange
 * shards by device copies with the NCCL collectives' semantics. */
#define XM_LOOPBACK_MAGIC "XM-LOOPBACK"
xm_status xm_create(xm_ctx** out, int device, int rank, int world, const void* nccl_id,
                    const xm_options* opts, void* cuda_stream);
void xm_destroy(xm_ctx* ctx);
xm_status xm_nccl_unique_id(void* out128);

/* Row shard of `rank` among `world` ranks.  Host-only: no
 * device work, callable without a GPU.  Rank q owns frames [*f0, *f1) ⇒ Q rows
 * [3·f0, 3·f1), and stores only their lower trapezoid (columns ≤ row): the
 * band layout that composes row sharding with the symmetric (lower-triangle)
 * stream.  Bands are contiguous, start at F_q = N·√(q/world) rounded to a
 * multiple of 32 frames (equal lower-triangle areas ⇒ equal Q bytes per
 * product on every rank); some may be empty.  *frames_per_rank (may be NULL)
 * = the largest band.  Each product is one all-reduce of the ranks' n×r
 * partials (row parts of the band, column parts above it).  XM_EINVAL on
 * N < 1, world < 1 or rank ∉ [0, world). */
xm_status xm_shard_rows(int32_t N, int32_t world, int32_t rank, int32_t* f0, int32_t* f1,
                        int32_t* frames_per_rank);

/* H1–H5.  Build Q from E observations (frame[e], landmark[e], ũ_e =
 * lifted_pts[3e..3e+2], w_e = weights[e] or 1 if weights == NULL).
 * Validates (XM_EINVAL), drops duplicate (frame, landmark) pairs keeping the
 * first (counted in xm_stats.n_dup), checks connectivity
 * (XM_EDISCONNECTED), then assembles Q = S − C̄ᵀ K̄⁻¹ C̄ on the device (Q rows
 * of this rank only). */
xm_status xm_build_Q(xm_ctx* ctx, int32_t N, int32_t M, int64_t E, const int32_t* frame,
                     const int32_t* landmark, const double* lifted_pts, const double* weights);

/* Algorithm 1 from U⁰ = [I₃,…,I₃] at r = r0 (r0 ≥ 3), or from the factor
 * set by xm_set_factor.  tol > 0 overrides opts.grad_tol.  Returns XM_OK if
 * certified, XM_UNCERTIFIED at the rank cap, XM_NOT_CONVERGED, or an error. */
xm_status xm_solve(xm_ctx* ctx, int32_t r0, double tol, xm_solve_info* info);

/* Certificate at the current factor (runs the Lanczos certificate and an
 * internal rounding to evaluate ρ̂ and η).  min_eigvec: n doubles or NULL. */
xm_status xm_certify(xm_ctx* ctx, xm_certificate* out, double* min_eigvec);

/* Rounded, gauge-fixed solution: R N×9 (row-major 3×3, camera→world), s N,
 * t N×3, p M×3 (NaN for landmarks with no observation); n_flipped = number of
 * blocks projected from det < 0 to SO(3).  Any output pointer may be NULL. */
xm_status xm_round_recover(xm_ctx* ctx, double* R, double* s, double* t, double* p,
                           int32_t* n_flipped);

/* ---------------------------------------------------------------- XM²
 * "delete the 10% measurements with the largest
 * residuals and re-run the XM solver … XM² (running twice)", with
 * SPEC's residual and never-disconnect rule;
 * selection / restoration order = reading C22.
 *
 * xm_edge_residuals: res[e] = w_e‖s_i R_i ũ_e + t_i − p_k‖² (the Eq. (3)
 *   summand) at the recovered solution of the last solve (rounds
 *   first if xm_round_recover was not called), for every measurement e of the
 *   caller's last xm_build_Q input, in that order (E doubles, host or device);
 *   NaN for duplicates and for measurements an XM² step dropped.  Requires a
 *   solve on a view graph (XM_ESTATE otherwise, or after xm_set_Q).
 * xm_xm2: rank the measurements in use by that residual (largest first,
 *   equal residuals by (landmark, frame) ascending), drop ⌊drop_fraction·E⌋,
 *   restore dropped ones smallest-residual-first where needed to keep the
 *   frames connected, and rebuild Q from the rest on the device.  The context
 *   returns to "Q built": call xm_solve / xm_certify / xm_round_recover again.
 *   keep (E bytes, caller's input order, host or device, or NULL): 1 for the
 *   measurements the rebuilt Q uses.  n_dropped / n_restored (or NULL): net
 *   drops and restorations.  drop_fraction ∉ [0, 1) ⇒ XM_EINVAL; a graph that
 *   no restoration reconnects ⇒ XM_EDISCONNECTED (context unchanged).  A
 *   failure while the rebuild replaces the data (e.g. XM_ENOMEM) leaves the
 *   context with no data (as after xm_create): rebuild with xm_build_Q.
 *   Repeated calls compose (indices always refer to the caller's original
 *   input). */
xm_status xm_edge_residuals(xm_ctx* ctx, double* res);
xm_status xm_xm2(xm_ctx* ctx, double drop_fraction, uint8_t* keep, int64_t* n_dropped,
                 int64_t* n_restored);

/* ------------------------------------------- batched small instances (NEXT-4) */
typedef struct {
  double f;               /* final objective ⟨Y, QY⟩                              */
  double grad_norm;
  double lambda_min;      /* λ_min(Z) by Lanczos (O6) at the final point          */
  double normQ;           /* ‖Q‖_F of the instance (tolerance scale)              */
  int32_t r;              /* final rank                                          */
  int32_t certified;
  int32_t status;         /* 0, XM_UNCERTIFIED, XM_NOT_CONVERGED, XM_ERETRACT,    */
                          /* XM_EESCAPE (per instance)                            */
  int32_t hvps;
  int32_t outer_iters;
  int32_t lanczos_steps;
} xm_batch_result;
/* B independent small instances, each the whole Algorithm 1 from
 * its own start — Thm 3's random-initialisation trials and App. G's
 * noise sweeps — in ONE launch: one CTA per instance (SURVEY
 * §8(f) NEXT-4); N ≤ 24: Q and all vectors in shared memory; 24 < N ≤ 400 (e.g.
 * the paper's BAL-93 trials): Q read from global memory (L2-resident when
 * shared), vectors in a per-instance device scratch.  Q: B matrices n×n
 * (row-major, n = 3N, caller memory, host or device), instance b at
 * Q + b·q_stride (q_stride = 0: one Q shared by every instance); Y0: B × n × r0
 * feasible starts; Y_out: B × n × 8 (row-major, stride 8, columns ≥ r zero);
 * res: B results.  Options (tolerances, TR / tCG constants, rank_cap ≤ 8,
 * seed) from the context; no App. D term.  Needs a context (for its device and
 * stream) but no xm_build_Q.  XM_EINVAL unless 1 ≤ N ≤ 400, 3 ≤ r0 ≤
 * min(rank_cap, 8), B ≥ 1.  Per-instance failures are reported in res, not as
 * the call's status. */
xm_status xm_solve_batch(xm_ctx* ctx, int32_t B, int32_t N, const double* Q, int64_t q_stride,
                         const double* Y0, int32_t r0, double* Y_out, xm_batch_result* res);

/* ----------------------------------------------------- test / bench hooks */
/* S's co-visibility BSR pattern (H3): rowptr N+1 (int64), colidx nnzb (int32,
 * sorted per row).  Call with colidx == NULL to query *nnzb. */
xm_status xm_get_S_pattern(xm_ctx* ctx, int64_t* rowptr, int32_t* colidx, int64_t* nnzb);
/* Rows [row0, row0+nrows) of Q (this rank must own them): nrows × n.  world > 1
 * after xm_build_Q: entries right of the diagonal are not stored (band
 * layout, xm_shard_rows) and come back as NaN. */
xm_status xm_get_Q_rows(xm_ctx* ctx, int32_t row0, int32_t nrows, double* out);
/* Replace Q by caller data (full n×n, row-major); this rank keeps its rows.
 * N is implied by n = 3N.  Allows parity tests on an identical Q. */
xm_status xm_set_Q(xm_ctx* ctx, int32_t N, const double* Q_full);
/* out (n×r) = Q·V (V: n×r). */
xm_status xm_spmm(xm_ctx* ctx, const double* V, double* out, int32_t r);
/* Riemannian gradient at Y (n×r): grad = P_Y(2QY); f = ⟨Y, QY⟩ (may be NULL). */
xm_status xm_grad(xm_ctx* ctx, const double* Y, double* grad, double* f, int32_t r);
/* Riemannian Hessian-vector product at Y along tangent V: P_Y(2QV − 2ΛV). */
xm_status xm_hvp(xm_ctx* ctx, const double* Y, const double* V, double* HV, int32_t r);
/* One Steihaug–Toint truncated-CG solve ("truncated conjugate
 * gradient") of the TR subproblem at Y (n×r,
 * caller memory, host or device): g = grad f(Y), Hess as xm_hvp, radius
 * Delta > 0, the context's κ / θ / max-inner options.  Outputs (caller
 * memory, n×r): eta = the step, Heta = Hess[eta] as accumulated by the
 * recurrence (may be NULL); *n_hvp = HVPs used; *stop = 1 negative curvature,
 * 2 boundary exceeded, 3 converged, 4 max inner.  path selects the device
 * implementation: 0 the library's choice, 1 persistent lower-triangle kernel
 * (k_tcg_persist_sym), 2 persistent full-row kernel (k_tcg_persist), 3 one
 * fused launch per iteration, 4 three kernels per iteration (CUDA graphs).
 * XM_EINVAL if that path is not available for (N, r).  Side effects: the
 * factor becomes Y (as xm_set_factor); certificate / rounding invalidated. */
xm_status xm_tcg(xm_ctx* ctx, const double* Y, int32_t r, double Delta, int32_t path, double* eta,
                 double* Heta, int32_t* n_hvp, int32_t* stop);
/* Tangent projection P_Y(W) and retraction R_Y(V). */
xm_status xm_project(xm_ctx* ctx, const double* Y, const double* W, double* out, int32_t r);
xm_status xm_retract(xm_ctx* ctx, const double* Y, const double* V, double* out, int32_t r);
/* Current factor (n×r; call with Y == NULL to query r) / warm start. */
xm_status xm_get_factor(xm_ctx* ctx, double* Y, int32_t* r);
xm_status xm_set_factor(xm_ctx* ctx, const double* Y, int32_t r);
xm_status xm_get_stats(xm_ctx* ctx, xm_stats* out);
xm_status xm_reset_stats(xm_ctx* ctx);
/* Switch per-launch CUDA-event timing of the Q·V kernels (xm_options.profile)
 * on or off for subsequent calls.  Event records inside the CUDA graphs cost
 * a few µs per launch, so timed runs that report the solve time keep it off
 * and a separate profiled run supplies the kernel timings. */
xm_status xm_set_profile(xm_ctx* ctx, int32_t on);
/* Human-readable detail of the last failed call on this context ("" if none;
 * the pointer stays valid until the next call). */
const char* xm_last_error(xm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* XM_H_ */
