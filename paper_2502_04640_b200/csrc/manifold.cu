// manifold.cu — per-camera kernels of the BM Riemannian solve (H7–H10, H12)
// and the device-resident truncated-CG iteration (H9).
//
// Manifold (Prop. 5): block 0 on St(r,3) (Y_0Y_0ᵀ = I), blocks
// i ≥ 1 on ℝ₊ × St(r,3) (Y_iY_iᵀ = α_i I).  Tangent vectors are ambient 3×r
// blocks with the Frobenius metric (reading C4).  One thread per camera: the
// whole 3×r block (r ≤ 12) lives in registers.
//
//   P_i(W)   = W − sym₀(W Y_iᵀ) Y_i / α_i        (i ≥ 1),   P_0(W) = W − sym(W Y_0ᵀ) Y_0
//   Λ_i      = sym₀((QY)_i Y_iᵀ)/α_i, Λ_0 = sym((QY)_0 Y_0ᵀ)  (Thm 1 Eq. (18), App. A.4)
//   grad     = 2(QY − ΛY)                                   (= P(2QY), reading C5)
//   Hess[V]  = P(2QV − 2ΛV)                                  (analytic HVP)
//   Retr     : s′ = max(s + ⟨V_i,R̂⟩/3, c·s), R̂′ = MGS(R̂ + W/s)   (C6, C7)
//   App. D (λ > 0, i ≥ 1, d_i = 2λ/3 (α_i − 1)):  f += λ(α_i − 1)²,
//     grad_i += 2 d_i Y_i,  Hess[V]_i += P_i(2 d_i V_i + 8λ/9 ⟨Y_i,V_i⟩ Y_i),  (ZX)_i += d_i X_i
//
// tCG (Steihaug–Toint in Manopt's form) runs as THREE kernels
// per iteration with the scalar recurrences folded in: every block recomputes
// the same scalar from the same partials in the same fixed order (so all blocks
// agree bit for bit), and block 0 writes the next state into the other half of
// a double-buffered TcgState — no host round trip, no separate control kernel:
//   K1  Hδ = Hess[δ] (SpMM + fused epilogue), partials of ⟨δ, Hδ⟩
//   K2  α, τ, boundary test; η += αδ, Hη += αHδ, r ← P(r + αHδ), partials ⟨r,r⟩
//   K3  stop tests, β, e_Pd/d_Pd recurrences; δ ← −r + βδ
#include "frame_ops.cuh"

namespace xm {

constexpr int kFT = 128;  // threads per block for per-frame kernels

// ------------------------------------------------------------------ H7 gradient
template <int R>
__global__ void __launch_bounds__(kFT) k_grad(int N, const double* __restrict__ Y,
                                              const double* __restrict__ QY,
                                              double* __restrict__ lam, double* __restrict__ grad,
                                              double* __restrict__ partials, double reg) {
  int i = blockIdx.x * kFT + threadIdx.x;
  double v[3] = {0.0, 0.0, 1.0e300};
  if (i < N) {
    Blk<R> y, g;
    load_blk<R>(Y, i, y);
    load_blk<R>(QY, i, g);
    double M[3][3], L[6];
    mul_abt<R>(g, y, M);
    double alpha = frob2<R>(y) / 3.0;
    sym_lambda(M, i == 0, alpha, L);
#pragma unroll
    for (int q = 0; q < 6; ++q) lam[6 * i + q] = L[q];
    Blk<R> gr;
    sub_lam<R>(g, L, y, 2.0, 2.0, gr);
    v[0] = dotb<R>(y, g);
    if (reg != 0.0 && i > 0) {  // App. D: radial (tangent) gradient 2 d_i Y_i, f += λ(α−1)²
      const double d = (2.0 * reg / 3.0) * (alpha - 1.0);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) gr.v[a][cc] = fma(2.0 * d, y.v[a][cc], gr.v[a][cc]);
      v[0] += reg * (alpha - 1.0) * (alpha - 1.0);
    }
    store_blk<R>(grad, i, gr);
    v[1] = frob2<R>(gr);
    if (i > 0) v[2] = alpha;
  }
  block_reduce_store<3, kFT>(v, partials, 4u);
}

// ------------------------------------------------------------------ projection
template <int R>
__global__ void __launch_bounds__(kFT) k_project(int N, const double* __restrict__ Y,
                                                 const double* __restrict__ W,
                                                 double* __restrict__ out) {
  int i = blockIdx.x * kFT + threadIdx.x;
  if (i >= N) return;
  Blk<R> y, w;
  load_blk<R>(Y, i, y);
  load_blk<R>(W, i, w);
  project_blk<R>(y, i == 0, w);
  store_blk<R>(out, i, w);
}

// ------------------------------------------------------------------ H8 HVP epilogue (unfused)
template <int R>
__global__ void __launch_bounds__(kFT) k_hvp(int N, const double* __restrict__ Y,
                                             const double* __restrict__ lam,
                                             const double* __restrict__ V,
                                             const double* __restrict__ QV,
                                             double* __restrict__ HV, double* __restrict__ partials,
                                             const int* __restrict__ stop, double reg) {
  if (stop && *stop) return;
  int i = blockIdx.x * kFT + threadIdx.x;
  double v[1] = {0.0};
  if (i < N) {
    Blk<R> y, vv, qv, w;
    load_blk<R>(Y, i, y);
    load_blk<R>(V, i, vv);
    load_blk<R>(QV, i, qv);
    double L[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) L[q] = lam[6 * i + q];
    sub_lam<R>(qv, L, vv, 2.0, 2.0, w);
    if (reg != 0.0 && i > 0) {  // App. D: + 2 d_i V_i + (8λ/9)⟨Y_i, V_i⟩ Y_i
      const double alpha = frob2<R>(y) / 3.0;
      const double d2 = 2.0 * (2.0 * reg / 3.0) * (alpha - 1.0);
      const double yv = (8.0 * reg / 9.0) * dotb<R>(y, vv);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int cc = 0; cc < R; ++cc)
          w.v[a][cc] = fma(d2, vv.v[a][cc], fma(yv, y.v[a][cc], w.v[a][cc]));
    }
    project_blk<R>(y, i == 0, w);
    store_blk<R>(HV, i, w);
    v[0] = dotb<R>(vv, w);
  }
  block_reduce_store<1, kFT>(v, partials);
}

// ------------------------------------------------------------------ H10 retraction
template <int R>
__global__ void __launch_bounds__(kFT) k_retract(int N, const double* __restrict__ Y,
                                                 const double* __restrict__ V, double step,
                                                 double c_floor, double* __restrict__ Yout,
                                                 double* __restrict__ D, int* __restrict__ err,
                                                 const double* __restrict__ g,
                                                 const double* __restrict__ HV,
                                                 double* __restrict__ dots2) {
  int i = blockIdx.x * kFT + threadIdx.x;
  double pd[2] = {0.0, 0.0};
  if (i < N) {
    Blk<R> y, v, m;
    load_blk<R>(Y, i, y);
    load_blk<R>(V, i, v);
    if (dots2) {
      Blk<R> gg, hv;
      load_blk<R>(g, i, gg);
      load_blk<R>(HV, i, hv);
      pd[0] = dotb<R>(gg, v);
      pd[1] = dotb<R>(v, hv);
    }
    double s_new;
    if (i == 0) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < R; ++c) m.v[a][c] = y.v[a][c] + step * v.v[a][c];
      s_new = 1.0;
    } else {
      double s = sqrt(frob2<R>(y) / 3.0);
      double is = 1.0 / s;
      double ds = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < R; ++c) ds = fma(step * v.v[a][c], y.v[a][c] * is, ds);
      ds /= 3.0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < R; ++c) {
          double rh = y.v[a][c] * is;
          double wt = step * v.v[a][c] - ds * rh;
          m.v[a][c] = rh + wt * is;
        }
      s_new = fmax(s + ds, c_floor * s);
    }
    // modified Gram–Schmidt on the three rows, positive diagonal (C20)
    double scale = sqrt(frob2<R>(m));
    bool bad = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int b = 0; b < a; ++b) {
        double d = 0.0;
#pragma unroll
        for (int c = 0; c < R; ++c) d = fma(m.v[a][c], m.v[b][c], d);
#pragma unroll
        for (int c = 0; c < R; ++c) m.v[a][c] -= d * m.v[b][c];
      }
      double nv = 0.0;
#pragma unroll
      for (int c = 0; c < R; ++c) nv = fma(m.v[a][c], m.v[a][c], nv);
      nv = sqrt(nv);
      if (!(nv > 1e-14 * scale)) {
        bad = true;
        nv = 1.0;
      }
      double inv = 1.0 / nv;
#pragma unroll
      for (int c = 0; c < R; ++c) m.v[a][c] *= inv;
    }
    if (bad) atomicOr(err, 1);
    Blk<R> out;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < R; ++c) out.v[a][c] = s_new * m.v[a][c];
    store_blk<R>(Yout, i, out);
    if (D) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < R; ++c) out.v[a][c] -= y.v[a][c];
      store_blk<R>(D, i, out);
    }
  }
  if (dots2) block_reduce_store<2, kFT>(pd, dots2);
}

// ------------------------------------------------------------------ H9 tCG
// Initialise: η = Hη = 0, r = g, δ = −g, state st[0] (z = ‖g‖² from the gradient pass).
__global__ void k_tcg_init_vec(int64_t len, const double* __restrict__ g, double* __restrict__ eta,
                               double* __restrict__ Heta, double* __restrict__ res,
                               double* __restrict__ dir) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= len) return;
  double gv = g[t];
  eta[t] = 0.0;
  Heta[t] = 0.0;
  res[t] = gv;
  dir[t] = -gv;
}
__global__ void k_tcg_init_state(TcgState* st, const double* __restrict__ z0, double Delta,
                                 double kappa, double theta, int max_inner) {
  TcgState s{};
  s.Delta = Delta;
  s.z = *z0;
  s.r0 = sqrt(s.z);
  s.d_Pd = s.z;
  s.kappa = kappa;
  s.theta = theta;
  s.max_inner = max_inner;
  s.stop = (max_inner <= 0) ? TCG_MAXINNER : TCG_RUNNING;
  st[0] = s;
  st[1] = s;
}

// K2: d_Hd from K1's partials; α, e_Pe′, boundary / τ; vector updates; ⟨r,r⟩ partials.
template <int R>
__global__ void __launch_bounds__(kFT) k_tcg_update(int N, const TcgState* __restrict__ sin,
                                                    TcgState* __restrict__ sout,
                                                    const double* __restrict__ p1, int n1,
                                                    const double* __restrict__ Y,
                                                    const double* __restrict__ dir,
                                                    const double* __restrict__ Hdir,
                                                    double* __restrict__ eta,
                                                    double* __restrict__ Heta,
                                                    double* __restrict__ res,
                                                    double* __restrict__ p2) {
  TcgState s = *sin;
  if (s.stop) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *sout = s;
    return;
  }
  const double dHd = block_sum_all<kFT>(p1, n1);
  s.d_Hd = dHd;
  s.n_hvp += 1;
  const double alpha = (dHd != 0.0) ? s.z / dHd : INFINITY;
  const double e_new = s.e_Pe + 2.0 * alpha * s.e_Pd + alpha * alpha * s.d_Pd;
  const double D2 = s.Delta * s.Delta;
  s.alpha = alpha;
  s.e_Pe_new = e_new;
  if (dHd <= 0.0 || e_new >= D2) {
    s.tau = (-s.e_Pd + sqrt(s.e_Pd * s.e_Pd + s.d_Pd * (D2 - s.e_Pe))) / s.d_Pd;
    s.boundary = 1;
    s.stop = (dHd <= 0.0) ? TCG_NEGCURV : TCG_EXCEEDED;
  } else {
    s.boundary = 0;
  }
  const double a = s.boundary ? s.tau : alpha;
  int i = blockIdx.x * kFT + threadIdx.x;
  double v[1] = {0.0};
  if (i < N) {
    Blk<R> d, hd, e, he;
    load_blk<R>(dir, i, d);
    load_blk<R>(Hdir, i, hd);
    load_blk<R>(eta, i, e);
    load_blk<R>(Heta, i, he);
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int c = 0; c < R; ++c) {
        e.v[p][c] = fma(a, d.v[p][c], e.v[p][c]);
        he.v[p][c] = fma(a, hd.v[p][c], he.v[p][c]);
      }
    store_blk<R>(eta, i, e);
    store_blk<R>(Heta, i, he);
    if (!s.boundary) {
      Blk<R> y, rr;
      load_blk<R>(Y, i, y);
      load_blk<R>(res, i, rr);
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int c = 0; c < R; ++c) rr.v[p][c] = fma(a, hd.v[p][c], rr.v[p][c]);
      project_blk<R>(y, i == 0, rr);
      store_blk<R>(res, i, rr);
      v[0] = frob2<R>(rr);
    }
  }
  block_reduce_store<1, kFT>(v, p2);
  if (blockIdx.x == 0 && threadIdx.x == 0) *sout = s;
}

// K3: stop tests, β, recurrences; δ ← −r + βδ.  Grid over n·r elements.
// cond ≠ 0: the kernel is the last node of the body of a conditional WHILE
// graph node (one graph launch runs the whole tCG loop, xm_api.cu tcg_graph):
// it clears the loop condition once the state says stop.
__global__ void __launch_bounds__(256) k_tcg_dir(int64_t len, const TcgState* __restrict__ sin,
                                                 TcgState* __restrict__ sout,
                                                 const double* __restrict__ p2, int n2,
                                                 const double* __restrict__ res,
                                                 double* __restrict__ dir,
                                                 cudaGraphConditionalHandle cond, int use_cond) {
  TcgState s = *sin;
  if (s.stop) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *sout = s;
      if (use_cond) cudaGraphSetConditional(cond, 0);
    }
    return;
  }
  const double z = block_sum_all<256>(p2, n2);
  s.e_Pe = s.e_Pe_new;
  s.z_old = s.z;
  s.z = z;
  s.j += 1;
  if (sqrt(z) <= s.r0 * fmin(pow(s.r0, s.theta), s.kappa)) {
    s.stop = TCG_CONVERGED;
  } else {
    s.beta = s.z / s.z_old;
    s.e_Pd = s.beta * (s.e_Pd + s.alpha * s.d_Pd);
    s.d_Pd = s.z + s.beta * s.beta * s.d_Pd;
    if (s.j >= s.max_inner) s.stop = TCG_MAXINNER;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *sout = s;
    if (use_cond && s.stop) cudaGraphSetConditional(cond, 0);
  }
  if (s.stop) return;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < len;
       t += (int64_t)gridDim.x * blockDim.x)
    dir[t] = fma(s.beta, dir[t], -res[t]);
}

// ------------------------------------------------------------------ misc vector ops
__global__ void k_axpy(int64_t len, double a, const double* __restrict__ x, double* __restrict__ y) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < len) y[t] = fma(a, x[t], y[t]);
}

// Yz = [Y, 0] (n × (r+1)), Dz = [0, v]
__global__ void k_pad_column(int64_t n, int r, const double* __restrict__ Y, double* __restrict__ Yz,
                             const double* __restrict__ v, double* __restrict__ Dz) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * (r + 1)) return;
  int64_t row = t / (r + 1);
  int c = (int)(t - row * (r + 1));
  Yz[t] = (c < r) ? Y[row * r + c] : 0.0;
  if (Dz) Dz[t] = (c < r) ? 0.0 : v[row];
}

// Zx = Qx − Λx for a single vector (r = 1), per camera
__global__ void __launch_bounds__(kFT) k_zmul(int N, const double* __restrict__ lam,
                                              const double* __restrict__ x,
                                              const double* __restrict__ qx,
                                              double* __restrict__ out,
                                              const double* __restrict__ regd) {
  int i = blockIdx.x * kFT + threadIdx.x;
  if (i >= N) return;
  double L[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) L[q] = lam[6 * i + q];
  if (regd) {  // Z_λ = Q + blkdiag(d_i I) − blkdiag(Λ)  (App. D)
    L[0] -= regd[i];
    L[1] -= regd[i];
    L[2] -= regd[i];
  }
  double x0 = x[3 * i], x1 = x[3 * i + 1], x2 = x[3 * i + 2];
  out[3 * i] = qx[3 * i] - (L[0] * x0 + L[3] * x1 + L[4] * x2);
  out[3 * i + 1] = qx[3 * i + 1] - (L[3] * x0 + L[1] * x1 + L[5] * x2);
  out[3 * i + 2] = qx[3 * i + 2] - (L[4] * x0 + L[5] * x1 + L[2] * x2);
}

// App. D per-frame helpers: d_i = 2λ/3 (α_i − 1) (d_0 = 0), and partial sums of
// λ(α_i−1)² [0], α_i² − 1 [1] over i ≥ 1, and of F(Y + D) − F(Y) computed
// without cancellation, λ(α′−α)(α′+α−2) with α′−α = ⟨D_i, 2Y_i + D_i⟩/3 [2]
template <int R>
__global__ void __launch_bounds__(kFT) k_reg_frames(int N, const double* __restrict__ Y,
                                                    const double* __restrict__ D, double reg,
                                                    double* __restrict__ regd,
                                                    double* __restrict__ partials) {
  int i = blockIdx.x * kFT + threadIdx.x;
  double v[3] = {0.0, 0.0, 0.0};
  if (i < N) {
    Blk<R> y;
    load_blk<R>(Y, i, y);
    const double alpha = frob2<R>(y) / 3.0;
    if (regd) regd[i] = (i > 0) ? (2.0 * reg / 3.0) * (alpha - 1.0) : 0.0;
    if (i > 0) {
      v[0] = reg * (alpha - 1.0) * (alpha - 1.0);
      v[1] = alpha * alpha - 1.0;
      if (D) {
        Blk<R> dd;
        load_blk<R>(D, i, dd);
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int cc = 0; cc < R; ++cc) s = fma(dd.v[a][cc], fma(2.0, y.v[a][cc], dd.v[a][cc]), s);
        const double da = s / 3.0;
        v[2] = reg * da * (2.0 * alpha + da - 2.0);
      }
    }
  }
  block_reduce_store<3, kFT>(v, partials);
}

// ================================================================== host wrappers
#define XM_DISPATCH_R(r, CALL)                                                      \
  switch (r) {                                                                      \
    case 1: { constexpr int R = 1; CALL; } break;                                   \
    case 2: { constexpr int R = 2; CALL; } break;                                   \
    case 3: { constexpr int R = 3; CALL; } break;                                   \
    case 4: { constexpr int R = 4; CALL; } break;                                   \
    case 5: { constexpr int R = 5; CALL; } break;                                   \
    case 6: { constexpr int R = 6; CALL; } break;                                   \
    case 7: { constexpr int R = 7; CALL; } break;                                   \
    case 8: { constexpr int R = 8; CALL; } break;                                   \
    case 9: { constexpr int R = 9; CALL; } break;                                   \
    case 10: { constexpr int R = 10; CALL; } break;                                 \
    case 11: { constexpr int R = 11; CALL; } break;                                 \
    case 12: { constexpr int R = 12; CALL; } break;                                 \
    default: throw Error(XM_EINVAL, "rank r out of range (1..12)");                \
  }

int frame_blocks(xm_ctx* c) { return ceil_div(c->N, kFT); }

void grad_and_multipliers(xm_ctx* c, int r, const double* Y, const double* QY, double* grad,
                          double* scal_out) {
  int nb = frame_blocks(c);
  c->red.alloc((size_t)nb * 4 + 1024);
  XM_DISPATCH_R(r, (k_grad<R><<<nb, kFT, 0, c->stream>>>(c->N, Y, QY, c->lam.p, grad, c->red.p,
                                                         c->opt.scale_reg)));
  XM_CHECK_LAUNCH();
  count_launch(c);
  reduce_partials(c, c->red.p, nb, 3, scal_out, 4u);
}

void project(xm_ctx* c, int r, const double* Y, const double* W, double* out) {
  XM_DISPATCH_R(r, (k_project<R><<<frame_blocks(c), kFT, 0, c->stream>>>(c->N, Y, W, out)));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void retract(xm_ctx* c, int r, const double* Y, const double* V, double step, double* Yout,
             double* D, int* err, const double* g, const double* HV, double* dots2) {
  XM_DISPATCH_R(r, (k_retract<R><<<frame_blocks(c), kFT, 0, c->stream>>>(
                       c->N, Y, V, step, c->opt.scale_floor, Yout, D, err, g, HV, dots2)));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void hvp_epilogue(xm_ctx* c, int r, const double* Y, const double* V, const double* QV,
                  double* HV, double* partials, const int* stop) {
  XM_DISPATCH_R(r, (k_hvp<R><<<frame_blocks(c), kFT, 0, c->stream>>>(c->N, Y, c->lam.p, V, QV, HV,
                                                                     partials, stop,
                                                                     c->opt.scale_reg)));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

int hvp_product(xm_ctx* c, int r, const double* Y, const double* V, double* HV, double* partials,
                const int* stop) {
  if (fused_epilogues(c)) {
    SpmmEpiArgs ep{};
    ep.Y = Y;
    ep.lam = c->lam.p;
    ep.out2 = HV;
    ep.partials = partials;
    ep.stop = stop;
    spmm(c, V, r, EPI_HVP, ep);
    return spmm_grid(c, r);
  }
  spmm_full(c, V, r, c->tmp.p, stop);
  hvp_epilogue(c, r, Y, V, c->tmp.p, HV, partials, stop);
  return frame_blocks(c);
}

void tcg_init(xm_ctx* c, int r, double Delta) {
  int64_t len = (int64_t)c->n * r;
  if (!c->gbar.p) {  // grid-barrier state of the fused kernels (never inside a capture)
    c->gbar.alloc(4);
    XM_CUDA(cudaMemsetAsync(c->gbar.p, 0, 4 * sizeof(int), c->stream));
  }
  c->gsync.alloc(4);
  XM_CUDA(cudaMemsetAsync(c->gsync.p, 0, 4 * sizeof(unsigned long long), c->stream));
  k_tcg_init_vec<<<ceil_div(len, 256), 256, 0, c->stream>>>(len, c->grad.p, c->eta.p, c->Heta.p,
                                                           c->res.p, c->dir.p);
  XM_CHECK_LAUNCH();
  // scal[1] holds ‖g‖² from the last gradient pass
  k_tcg_init_state<<<1, 1, 0, c->stream>>>(c->tcg.p, c->scal.p + 1, Delta, c->opt.tcg_kappa,
                                           c->opt.tcg_theta, c->opt.tcg_max_inner);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
}

// One tCG iteration.  One GPU, full-row SpMM: ONE cooperative launch
// (Q·δ → Hδ → grid barrier → α, η, Hη, r → grid barrier → β, δ; spmm.cu
// EPI_TCG), state st[0] → st[0].  Otherwise three kernels, st[0] → st[1] → st[0].
void tcg_iteration(xm_ctx* c, int r) {
  const int nb = frame_blocks(c);
  const int64_t len = (int64_t)c->n * r;
  c->part1.alloc(2048);
  c->part2.alloc((size_t)nb + 4096);
  if (tcg_fused_supported(c, r)) {
    SpmmEpiArgs ep{};
    ep.out = c->dir.p;
    ep.Y = c->Y.p;
    ep.lam = c->lam.p;
    ep.partials = c->part1.p;
    ep.stop = &c->tcg.p[0].stop;
    ep.st = c->tcg.p;
    ep.eta = c->eta.p;
    ep.Heta = c->Heta.p;
    ep.res = c->res.p;
    ep.p2 = c->part2.p;
    ep.gbar = reinterpret_cast<GridBar*>(c->gbar.p);
    ep.gsync = c->gsync.p;
    ep.out2 = c->Hdir.p;  // Q·δ rows (row-balanced producers → camera-owned consumers)
    if (c->phases_on) {
      if (!c->tdbg.p) {
        c->tdbg.alloc(148 * 8);
        XM_CUDA(cudaMemsetAsync(c->tdbg.p, 0, 148 * 8 * 8, c->stream));
      }
      ep.dbg = c->tdbg.p;
    }
    spmm(c, c->dir.p, r, EPI_TCG, ep);
    return;
  }
  int n1 = hvp_product(c, r, c->Y.p, c->dir.p, c->Hdir.p, c->part1.p, &c->tcg.p[0].stop);
  XM_DISPATCH_R(r, (k_tcg_update<R><<<nb, kFT, 0, c->stream>>>(
                       c->N, c->tcg.p, c->tcg.p + 1, c->part1.p, n1, c->Y.p, c->dir.p, c->Hdir.p,
                       c->eta.p, c->Heta.p, c->res.p, c->part2.p)));
  XM_CHECK_LAUNCH();
  int g3 = std::max(1, std::min(ceil_div(len, 256), 148));
  k_tcg_dir<<<g3, 256, 0, c->stream>>>(len, c->tcg.p + 1, c->tcg.p, c->part2.p, nb, c->res.p,
                                       c->dir.p, c->cap_cond, c->cap_cond_on ? 1 : 0);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
}

void axpy(xm_ctx* c, int64_t len, double a, const double* x, double* y) {
  k_axpy<<<ceil_div(len, 256), 256, 0, c->stream>>>(len, a, x, y);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void pad_column(xm_ctx* c, int r, const double* Y, double* Yz, const double* v, double* Dz) {
  int64_t len = (int64_t)c->n * (r + 1);
  k_pad_column<<<ceil_div(len, 256), 256, 0, c->stream>>>(c->n, r, Y, Yz, v, Dz);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

// App. D sums at Y (and F(Y + D) − F(Y) if D): scal_out[0] = F(Y), [1] = Σ_{i≥1}(α_i²−1),
// [2] = ΔF; d_i into c->regd.
void reg_frames(xm_ctx* c, int r, const double* Y, const double* D, double* scal_out) {
  const int nb = frame_blocks(c);
  c->regd.alloc((size_t)c->N + 8);
  DBuf<double>& part = scratch_f64(c, "reg_part");
  part.alloc((size_t)nb * 3 + 8);
  XM_DISPATCH_R(r, (k_reg_frames<R><<<nb, kFT, 0, c->stream>>>(c->N, Y, D, c->opt.scale_reg,
                                                              c->regd.p, part.p)));
  XM_CHECK_LAUNCH();
  count_launch(c);
  reduce_partials(c, part.p, nb, 3, scal_out);
}

void zmul(xm_ctx* c, const double* x, const double* Zx_q, double* out) {
  k_zmul<<<frame_blocks(c), kFT, 0, c->stream>>>(c->N, c->lam.p, x, Zx_q, out,
                                                 c->opt.scale_reg != 0.0 ? c->regd.p : nullptr);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

}  // namespace xm
