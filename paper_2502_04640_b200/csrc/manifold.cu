// manifold.cu — per-camera kernels of the BM Riemannian solve (H7–H10, H12).
//
// Manifold (Prop. 5): block 0 on St(r,3) (Y_0Y_0ᵀ = I), blocks
// i ≥ 1 on ℝ₊ × St(r,3) (Y_iY_iᵀ = α_i I).  Tangent vectors are ambient 3×r
// blocks with the Frobenius metric (reading C4).  One thread per camera: the
// whole 3×r block (r ≤ 12) lives in registers; the r×r-free formulas below only
// need the 3×3 matrix M = W Y_iᵀ.
//
//   P_i(W)   = W − sym₀(W Y_iᵀ) Y_i / α_i        (i ≥ 1),   P_0(W) = W − sym(W Y_0ᵀ) Y_0
//   Λ_i      = sym₀((QY)_i Y_iᵀ)/α_i, Λ_0 = sym((QY)_0 Y_0ᵀ)  (Thm 1 Eq. (18), App. A.4)
//   grad     = 2(QY − ΛY)                                   (= P(2QY), reading C5)
//   Hess[V]  = P(2QV − 2ΛV)                                  (analytic HVP)
//   Retr     : s′ = max(s + ⟨V_i,R̂⟩/3, c·s), R̂′ = MGS(R̂ + W/s)   (C6, C7)
//
// Sums (dots) are reduced deterministically: per-thread camera sums → fixed
// block tree → per-block partials → one fixed-order final block.
#include "xm_internal.cuh"

namespace xm {

constexpr int kFT = 128;  // threads per block for per-frame kernels

template <int R>
struct Blk {
  double v[3][R];
};

template <int R>
__device__ __forceinline__ void load_blk(const double* __restrict__ X, int i, Blk<R>& b) {
  const double* p = X + (int64_t)3 * i * R;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) b.v[a][c] = p[a * R + c];
}
template <int R>
__device__ __forceinline__ void store_blk(double* __restrict__ X, int i, const Blk<R>& b) {
  double* p = X + (int64_t)3 * i * R;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) p[a * R + c] = b.v[a][c];
}
// M = A Bᵀ (3×3)
template <int R>
__device__ __forceinline__ void mul_abt(const Blk<R>& A, const Blk<R>& B, double M[3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < R; ++c) s = fma(A.v[a][c], B.v[b][c], s);
      M[a][b] = s;
    }
}
template <int R>
__device__ __forceinline__ double frob2(const Blk<R>& A) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) s = fma(A.v[a][c], A.v[a][c], s);
  return s;
}
template <int R>
__device__ __forceinline__ double dotb(const Blk<R>& A, const Blk<R>& B) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) s = fma(A.v[a][c], B.v[a][c], s);
  return s;
}
// Λ = sym(M) (anchor) or sym₀(M)/α, stored as (xx, yy, zz, xy, xz, yz)
__device__ __forceinline__ void sym_lambda(const double M[3][3], bool anchor, double alpha,
                                           double L[6]) {
  double xx = M[0][0], yy = M[1][1], zz = M[2][2];
  double xy = 0.5 * (M[0][1] + M[1][0]);
  double xz = 0.5 * (M[0][2] + M[2][0]);
  double yz = 0.5 * (M[1][2] + M[2][1]);
  if (anchor) {
    L[0] = xx; L[1] = yy; L[2] = zz; L[3] = xy; L[4] = xz; L[5] = yz;
  } else {
    double tr3 = (xx + yy + zz) / 3.0;
    double ia = 1.0 / alpha;
    L[0] = (xx - tr3) * ia; L[1] = (yy - tr3) * ia; L[2] = (zz - tr3) * ia;
    L[3] = xy * ia; L[4] = xz * ia; L[5] = yz * ia;
  }
}
// out = A − Λ B   (Λ symmetric 3×3 in packed form)
template <int R>
__device__ __forceinline__ void sub_lam(const Blk<R>& A, const double L[6], const Blk<R>& B,
                                        double scaleA, double scaleL, Blk<R>& out) {
  const double Lm[3][3] = {{L[0], L[3], L[4]}, {L[3], L[1], L[5]}, {L[4], L[5], L[2]}};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double s = Lm[a][0] * B.v[0][c] + Lm[a][1] * B.v[1][c] + Lm[a][2] * B.v[2][c];
      out.v[a][c] = scaleA * A.v[a][c] - scaleL * s;
    }
}
// in-place tangent projection of W at Y
template <int R>
__device__ __forceinline__ void project_blk(const Blk<R>& Y, bool anchor, Blk<R>& W) {
  double M[3][3], L[6];
  mul_abt<R>(W, Y, M);
  double alpha = anchor ? 1.0 : frob2<R>(Y) / 3.0;
  sym_lambda(M, anchor, alpha, L);
  Blk<R> o;
  sub_lam<R>(W, L, Y, 1.0, 1.0, o);
  W = o;
}

// block reduce of NC components → partials[blockIdx.x * NC + c]
template <int NC>
__device__ __forceinline__ void block_reduce_store(double (&v)[NC], double* __restrict__ partials,
                                                   const bool* is_min = nullptr) {
  __shared__ double sh[NC][kFT];
#pragma unroll
  for (int c = 0; c < NC; ++c) sh[c][threadIdx.x] = v[c];
  __syncthreads();
  for (int s = kFT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double a = sh[c][threadIdx.x], b = sh[c][threadIdx.x + s];
        sh[c][threadIdx.x] = (is_min && is_min[c]) ? fmin(a, b) : a + b;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) partials[blockIdx.x * NC + c] = sh[c][0];
  }
}

// ------------------------------------------------------------------ H7 gradient
template <int R>
__global__ void __launch_bounds__(kFT) k_grad(int N, const double* __restrict__ Y,
                                              const double* __restrict__ QY,
                                              double* __restrict__ lam, double* __restrict__ grad,
                                              double* __restrict__ partials) {
  int i = blockIdx.x * kFT + threadIdx.x;
  double v[3] = {0.0, 0.0, 1.0e300};
  if (i < N) {
    Blk<R> y, g;
    load_blk<R>(Y, i, y);
    load_blk<R>(QY, i, g);
    double M[3][3], L[6];
    mul_abt<R>(g, y, M);
    double a2 = frob2<R>(y);
    double alpha = a2 / 3.0;
    sym_lambda(M, i == 0, alpha, L);
#pragma unroll
    for (int q = 0; q < 6; ++q) lam[6 * i + q] = L[q];
    Blk<R> gr;
    sub_lam<R>(g, L, y, 2.0, 2.0, gr);
    store_blk<R>(grad, i, gr);
    v[0] = dotb<R>(y, g);
    v[1] = frob2<R>(gr);
    if (i > 0) v[2] = alpha;
  }
  const bool mins[3] = {false, false, true};
  block_reduce_store<3>(v, partials, mins);
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

// ------------------------------------------------------------------ H8 HVP epilogue
template <int R>
__global__ void __launch_bounds__(kFT) k_hvp(int N, const double* __restrict__ Y,
                                             const double* __restrict__ lam,
                                             const double* __restrict__ V,
                                             const double* __restrict__ QV,
                                             double* __restrict__ HV, double* __restrict__ partials,
                                             const int* __restrict__ stop) {
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
    sub_lam<R>(qv, L, vv, 2.0, 2.0, w);  // 2QV − 2ΛV
    project_blk<R>(y, i == 0, w);
    store_blk<R>(HV, i, w);
    v[0] = dotb<R>(vv, w);
  }
  block_reduce_store<1>(v, partials);
}

// ------------------------------------------------------------------ H10 retraction
template <int R>
__global__ void __launch_bounds__(kFT) k_retract(int N, const double* __restrict__ Y,
                                                 const double* __restrict__ V, double step,
                                                 double c_floor, double* __restrict__ Yout,
                                                 double* __restrict__ D, int* __restrict__ err) {
  int i = blockIdx.x * kFT + threadIdx.x;
  if (i >= N) return;
  Blk<R> y, v, m;
  load_blk<R>(Y, i, y);
  load_blk<R>(V, i, v);
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

// ------------------------------------------------------------------ H9 tCG (device state)
// Initialise: η = Hη = 0, r = g, δ = −g, z = ⟨r, r⟩ (from the gradient pass).
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
  s.e_Pe = 0.0;
  s.e_Pd = 0.0;
  s.d_Pd = s.z;
  s.kappa = kappa;
  s.theta = theta;
  s.max_inner = max_inner;
  s.stop = (max_inner <= 0) ? TCG_MAXINNER : TCG_RUNNING;
  *st = s;
}

// fixed-order sum of block partials inside a single 256-thread block
__device__ __forceinline__ double block_sum_partials(const double* __restrict__ part, int nblk) {
  __shared__ double sh[256];
  double a = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) a += part[b];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

// after the HVP: d_Hd, α, boundary test (Manopt / Steihaug–Toint, O5)
__global__ void __launch_bounds__(256) k_tcg_ctrl_a(TcgState* st, const double* __restrict__ part,
                                                    int nblk) {
  if (st->stop) return;
  double dHd = block_sum_partials(part, nblk);
  if (threadIdx.x != 0) return;
  TcgState s = *st;
  s.d_Hd = dHd;
  s.n_hvp += 1;
  double alpha = (dHd != 0.0) ? s.z / dHd : INFINITY;
  double e_new = s.e_Pe + 2.0 * alpha * s.e_Pd + alpha * alpha * s.d_Pd;
  s.alpha = alpha;
  s.e_Pe_new = e_new;
  double D2 = s.Delta * s.Delta;
  if (dHd <= 0.0 || e_new >= D2) {
    s.tau = (-s.e_Pd + sqrt(s.e_Pd * s.e_Pd + s.d_Pd * (D2 - s.e_Pe))) / s.d_Pd;
    s.boundary = 1;
  } else {
    s.boundary = 0;
  }
  *st = s;
}

template <int R>
__global__ void __launch_bounds__(kFT) k_tcg_update(int N, const TcgState* __restrict__ st,
                                                    const double* __restrict__ Y,
                                                    const double* __restrict__ dir,
                                                    const double* __restrict__ Hdir,
                                                    double* __restrict__ eta,
                                                    double* __restrict__ Heta,
                                                    double* __restrict__ res,
                                                    double* __restrict__ partials) {
  if (st->stop) return;
  const int boundary = st->boundary;
  const double a = boundary ? st->tau : st->alpha;
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
    if (!boundary) {
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
  block_reduce_store<1>(v, partials);
}

// after the update: stop tests, β, e_Pd / d_Pd recurrences
__global__ void __launch_bounds__(256) k_tcg_ctrl_b(TcgState* st, const double* __restrict__ part,
                                                    int nblk) {
  if (st->stop) return;
  double z = block_sum_partials(part, nblk);
  if (threadIdx.x != 0) return;
  TcgState s = *st;
  if (s.boundary) {
    s.stop = (s.d_Hd <= 0.0) ? TCG_NEGCURV : TCG_EXCEEDED;
    *st = s;
    return;
  }
  s.e_Pe = s.e_Pe_new;
  s.z_old = s.z;
  s.z = z;
  s.j += 1;
  double rn = sqrt(z);
  if (rn <= s.r0 * fmin(pow(s.r0, s.theta), s.kappa)) {
    s.stop = TCG_CONVERGED;
  } else {
    s.beta = s.z / s.z_old;
    s.e_Pd = s.beta * (s.e_Pd + s.alpha * s.d_Pd);
    s.d_Pd = s.z + s.beta * s.beta * s.d_Pd;
    if (s.j >= s.max_inner) s.stop = TCG_MAXINNER;
  }
  *st = s;
}

__global__ void k_tcg_dir(int64_t len, const TcgState* __restrict__ st,
                          const double* __restrict__ res, double* __restrict__ dir) {
  if (st->stop) return;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= len) return;
  dir[t] = fma(st->beta, dir[t], -res[t]);
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
                                              double* __restrict__ out) {
  int i = blockIdx.x * kFT + threadIdx.x;
  if (i >= N) return;
  double L[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) L[q] = lam[6 * i + q];
  double x0 = x[3 * i], x1 = x[3 * i + 1], x2 = x[3 * i + 2];
  out[3 * i] = qx[3 * i] - (L[0] * x0 + L[3] * x1 + L[4] * x2);
  out[3 * i + 1] = qx[3 * i + 1] - (L[3] * x0 + L[1] * x1 + L[5] * x2);
  out[3 * i + 2] = qx[3 * i + 2] - (L[4] * x0 + L[5] * x1 + L[2] * x2);
}

template <int R>
__global__ void __launch_bounds__(kFT) k_min_alpha(int N, const double* __restrict__ Y,
                                                   double* __restrict__ partials) {
  int i = blockIdx.x * kFT + threadIdx.x;
  double v[1] = {1.0e300};
  if (i > 0 && i < N) {
    Blk<R> y;
    load_blk<R>(Y, i, y);
    v[0] = frob2<R>(y) / 3.0;
  }
  const bool mins[1] = {true};
  block_reduce_store<1>(v, partials, mins);
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

static inline int fblocks(int N) { return ceil_div(N, kFT); }

void grad_and_multipliers(xm_ctx* c, int r, const double* Y, const double* QY, double* grad,
                          double* scal_out) {
  int nb = fblocks(c->N);
  c->red.alloc((size_t)nb * 4 + 1024);
  XM_DISPATCH_R(r, (k_grad<R><<<nb, kFT, 0, c->stream>>>(c->N, Y, QY, c->lam.p, grad, c->red.p)));
  XM_CHECK_LAUNCH();
  count_launch(c);
  reduce_partials(c, c->red.p, nb, 3, scal_out, 4u);
}

void project(xm_ctx* c, int r, const double* Y, const double* W, double* out) {
  XM_DISPATCH_R(r, (k_project<R><<<fblocks(c->N), kFT, 0, c->stream>>>(c->N, Y, W, out)));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void retract(xm_ctx* c, int r, const double* Y, const double* V, double step, double* Yout,
             double* D, int* err) {
  XM_DISPATCH_R(r, (k_retract<R><<<fblocks(c->N), kFT, 0, c->stream>>>(
                       c->N, Y, V, step, c->opt.scale_floor, Yout, D, err)));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void hvp_epilogue(xm_ctx* c, int r, const double* Y, const double* V, const double* QV,
                  double* HV, double* dot_out, const int* stop) {
  int nb = fblocks(c->N);
  c->red.alloc((size_t)nb * 4 + 1024);
  XM_DISPATCH_R(r, (k_hvp<R><<<nb, kFT, 0, c->stream>>>(c->N, Y, c->lam.p, V, QV, HV, c->red.p,
                                                        stop)));
  XM_CHECK_LAUNCH();
  count_launch(c);
  if (dot_out) reduce_partials(c, c->red.p, nb, 1, dot_out);
}

void tcg_init(xm_ctx* c, int r, double Delta) {
  int64_t len = (int64_t)c->n * r;
  k_tcg_init_vec<<<ceil_div(len, 256), 256, 0, c->stream>>>(len, c->grad.p, c->eta.p, c->Heta.p,
                                                           c->res.p, c->dir.p);
  XM_CHECK_LAUNCH();
  // scal[1] holds ‖g‖² from the last gradient pass
  k_tcg_init_state<<<1, 1, 0, c->stream>>>(c->tcg.p, c->scal.p + 1, Delta, c->opt.tcg_kappa,
                                           c->opt.tcg_theta, c->opt.tcg_max_inner);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
}

void tcg_ctrl_a(xm_ctx* c) {
  k_tcg_ctrl_a<<<1, 256, 0, c->stream>>>(c->tcg.p, c->red.p, fblocks(c->N));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void tcg_update(xm_ctx* c, int r) {
  int nb = fblocks(c->N);
  XM_DISPATCH_R(r, (k_tcg_update<R><<<nb, kFT, 0, c->stream>>>(c->N, c->tcg.p, c->Y.p, c->dir.p,
                                                               c->Hdir.p, c->eta.p, c->Heta.p,
                                                               c->res.p, c->red.p)));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void tcg_ctrl_b(xm_ctx* c) {
  k_tcg_ctrl_b<<<1, 256, 0, c->stream>>>(c->tcg.p, c->red.p, fblocks(c->N));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void tcg_dir(xm_ctx* c, int r) {
  int64_t len = (int64_t)c->n * r;
  k_tcg_dir<<<ceil_div(len, 256), 256, 0, c->stream>>>(len, c->tcg.p, c->res.p, c->dir.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
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

void zmul(xm_ctx* c, const double* x, const double* Zx_q, double* out) {
  k_zmul<<<fblocks(c->N), kFT, 0, c->stream>>>(c->N, c->lam.p, x, Zx_q, out);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

double min_scale(xm_ctx* c, int r, const double* Y) {
  int nb = fblocks(c->N);
  c->red.alloc((size_t)nb * 4 + 1024);
  XM_DISPATCH_R(r, (k_min_alpha<R><<<nb, kFT, 0, c->stream>>>(c->N, Y, c->red.p)));
  XM_CHECK_LAUNCH();
  count_launch(c);
  reduce_partials(c, c->red.p, nb, 1, c->scal.p + 40, 1u);
  double a = 0.0;
  XM_CUDA(cudaMemcpyAsync(&a, c->scal.p + 40, 8, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  return c->N > 1 ? sqrt(a) : 1.0;
}

}  // namespace xm
