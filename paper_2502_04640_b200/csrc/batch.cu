// batch.cu — SURVEY §8(f) NEXT-4: many small instances solved at once
// (Thm 3's random-initialisation trials, "1000 trials"; App. G's noise
// sweep).  One CTA per instance runs the WHOLE Algorithm 1
// in shared memory — the RTR outer loop (O4) with its
// Steihaug–Toint tCG (O5), the retraction (C6, C7), the Lanczos certificate
// with full re-orthogonalisation (O6, C19) and the staircase escape (O7, C9)
// — with the same constants and formulas as the single-instance path and the
// oracle, so a batch of B instances is ONE launch of B CTAs instead of B
// latency-bound solves of hundreds of tiny kernels each.
//
// Layout: every n × r array is stored n × kBR (kBR = 8 columns, row stride 8);
// columns ≥ r are exactly zero and stay zero under every operation (products,
// multipliers, projection, retraction, escapes add column r), so the rank is
// implicit and the staircase never re-lays memory out.  n ≤ 72 (N ≤ 24):
// Q (41 KB), 12 vectors (55 KB) and the Lanczos basis (41 KB) fit in shared
// memory.  Reductions are fixed-order block trees (deterministic).
#include "frame_ops.cuh"

#include <cmath>

namespace xm {

namespace {
constexpr int kBT = 256;   // threads per instance
constexpr int kBR = 8;     // column stride (max rank)
constexpr int kBNmax = 24; // frames per instance with everything in shared memory
constexpr int kBNmaxGM = 400;  // frames per instance in the global-memory layout

struct BatchArgs {
  int B, N, n, r0, rcap;
  const double* Q;
  int64_t qstride;
  const double* Y0;
  double* Yout;
  xm_batch_result* res;
  double grad_tol, delta0_coef, delta_max_mult, rho_prime, kappa, theta, eig_tol, cert_tol, c_floor;
  int max_inner, max_outer, refresh_every, lanczos_max;
  uint64_t seed;
  double* scratch;         // GM layout: per-instance vectors / Lanczos basis in global memory
  int64_t scratch_stride;  // doubles per instance
};

struct Sm {
  double* Q;
  double *Y, *QY, *G, *ETA, *HETA, *RR, *DEL, *HDEL, *TMP, *YN, *DD, *QD;
  double* LAM;   // N × 6
  double* V;     // Lanczos basis, rows of n
  double* w;     // n
  double* al;    // alphas
  double* be;    // betas
  double* sv;    // Ritz vector coefficients
  double* red;   // kBT
  double* scal;  // broadcast scalars
};

__device__ double bsum(double x, double* red) {
  red[threadIdx.x] = x;
  __syncthreads();
  for (int s = kBT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double v = red[0];
  __syncthreads();
  return v;
}
__device__ double bdot(const double* a, const double* b, int len, double* red) {
  double s = 0.0;
  for (int x = threadIdx.x; x < len; x += kBT) s = fma(a[x], b[x], s);
  return bsum(s, red);
}
// out (n × 8) = Q (n × n) · X (n × 8) for the rc leading columns (the others of X
// are zero, so are those of out)
__device__ void bmatvec(const double* Q, int n, const double* X, double* out, int rc) {
  for (int e = threadIdx.x; e < n * rc; e += kBT) {
    const int row = e / rc, c = e - row * rc;
    const double* q = Q + (int64_t)row * n;
    double s = 0.0;
    for (int k = 0; k < n; ++k) s = fma(q[k], X[k * kBR + c], s);
    out[row * kBR + c] = s;
  }
  for (int e = threadIdx.x; e < n * (kBR - rc); e += kBT) {
    const int row = e / (kBR - rc), c = rc + (e - row * (kBR - rc));
    out[row * kBR + c] = 0.0;
  }
  __syncthreads();
}
// Λ_i from (QY)_i, Y_i (Thm 1 Eq. (18): sym₀(·)/α_i, anchor sym)
__device__ void bmult(const double* Y, const double* QY, double* LAM, int N) {
  const int i = threadIdx.x;
  if (i < N) {
    double M[3][3], yy = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int c = 0; c < kBR; ++c) s = fma(QY[(3 * i + a) * kBR + c], Y[(3 * i + b) * kBR + c], s);
        M[a][b] = s;
      }
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < kBR; ++c) yy = fma(Y[(3 * i + a) * kBR + c], Y[(3 * i + a) * kBR + c], yy);
    sym_lambda(M, i == 0, yy / 3.0, LAM + 6 * i);
  }
  __syncthreads();
}
__device__ __forceinline__ double lam_at(const double* L, int a, int b) {
  const int idx[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
  return L[idx[a][b]];
}
// out = sA·A − sL·blkdiag(Λ)·B
__device__ void bsublam(const double* A, const double* LAM, const double* Bm, double sA, double sL,
                        double* out, int n) {
  for (int e = threadIdx.x; e < n * kBR; e += kBT) {
    const int row = e / kBR, c = e % kBR, i = row / 3, a = row % 3;
    const double* L = LAM + 6 * i;
    double s = 0.0;
    for (int b = 0; b < 3; ++b) s = fma(lam_at(L, a, b), Bm[(3 * i + b) * kBR + c], s);
    out[e] = sA * A[e] - sL * s;
  }
  __syncthreads();
}
// in-place tangent projection P_Y(W) per frame (reading C4)
__device__ void bproject(const double* Y, double* W, int N) {
  const int i = threadIdx.x;
  if (i < N) {
    double M[3][3], yy = 0.0, L[6];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int c = 0; c < kBR; ++c) s = fma(W[(3 * i + a) * kBR + c], Y[(3 * i + b) * kBR + c], s);
        M[a][b] = s;
      }
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < kBR; ++c) yy = fma(Y[(3 * i + a) * kBR + c], Y[(3 * i + a) * kBR + c], yy);
    sym_lambda(M, i == 0, yy / 3.0, L);
    double o[3][kBR];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < kBR; ++c) {
        double s = 0.0;
        for (int b = 0; b < 3; ++b) s = fma(lam_at(L, a, b), Y[(3 * i + b) * kBR + c], s);
        o[a][c] = W[(3 * i + a) * kBR + c] - s;
      }
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < kBR; ++c) W[(3 * i + a) * kBR + c] = o[a][c];
  }
  __syncthreads();
}
// Hess[V] = P(2QV − 2ΛV) (reading C5) → out
__device__ void bhess(const Sm& s, const double* V, double* out, int n, int N, int rc) {
  bmatvec(s.Q, n, V, s.TMP, rc);
  bsublam(s.TMP, s.LAM, V, 2.0, 2.0, out, n);
  bproject(s.Y, out, N);
}
// retraction (C6, C7): Yout = R_Y(step·V), D = Yout − Y; returns 1 on a GS breakdown
__device__ int bretract(const double* Y, const double* V, double step, double c_floor, double* Yout,
                        double* D, int N, double* red) {
  const int i = threadIdx.x;
  int bad = 0;
  if (i < N) {
    double y[3][kBR], m[3][kBR], s_new;
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < kBR; ++c) y[a][c] = Y[(3 * i + a) * kBR + c];
    if (i == 0) {
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < kBR; ++c) m[a][c] = y[a][c] + step * V[(3 * i + a) * kBR + c];
      s_new = 1.0;
    } else {
      double f2 = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < kBR; ++c) f2 = fma(y[a][c], y[a][c], f2);
      const double sc = sqrt(f2 / 3.0), is = 1.0 / sc;
      double ds = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < kBR; ++c) ds = fma(step * V[(3 * i + a) * kBR + c], y[a][c] * is, ds);
      ds /= 3.0;
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < kBR; ++c) {
          const double rh = y[a][c] * is;
          const double wt = step * V[(3 * i + a) * kBR + c] - ds * rh;
          m[a][c] = rh + wt * is;
        }
      s_new = fmax(sc + ds, c_floor * sc);
    }
    double f2 = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < kBR; ++c) f2 = fma(m[a][c], m[a][c], f2);
    const double scale = sqrt(f2);
    for (int a = 0; a < 3; ++a) {  // modified Gram–Schmidt, positive diagonal (C20)
      for (int b = 0; b < a; ++b) {
        double d = 0.0;
        for (int c = 0; c < kBR; ++c) d = fma(m[a][c], m[b][c], d);
        for (int c = 0; c < kBR; ++c) m[a][c] -= d * m[b][c];
      }
      double nv = 0.0;
      for (int c = 0; c < kBR; ++c) nv = fma(m[a][c], m[a][c], nv);
      nv = sqrt(nv);
      if (!(nv > 1e-14 * scale)) {
        bad = 1;
        nv = 1.0;
      }
      const double inv = 1.0 / nv;
      for (int c = 0; c < kBR; ++c) m[a][c] *= inv;
    }
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < kBR; ++c) {
        const double o = s_new * m[a][c];
        Yout[(3 * i + a) * kBR + c] = o;
        if (D) D[(3 * i + a) * kBR + c] = o - y[a][c];
      }
  }
  __syncthreads();
  return bsum((double)bad, red) > 0.0 ? 1 : 0;
}

// smallest eigenpair of the symmetric tridiagonal (a[0..k), b[0..k−1)) — Sturm
// bisection + inverse iteration, one thread (as cert.cu's tridiag_min)
__device__ int sturm(const double* a, const double* b, int k, double x) {
  int cnt = 0;
  double d = a[0] - x;
  if (d < 0) ++cnt;
  for (int i = 1; i < k; ++i) {
    if (d == 0.0) d = 1e-300;
    d = a[i] - x - b[i - 1] * b[i - 1] / d;
    if (d < 0) ++cnt;
  }
  return cnt;
}
__device__ void tri_min(const double* a, const double* b, int k, double* lam, double* s, double* wk) {
  if (k == 1) {
    *lam = a[0];
    s[0] = 1.0;
    return;
  }
  double lo = a[0], hi = a[0];
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < k - 1 ? fabs(b[i]) : 0.0);
    lo = fmin(lo, a[i] - r);
    hi = fmax(hi, a[i] + r);
  }
  const double span = fmax(hi - lo, 1e-300);
  for (int it = 0; it < 200 && hi - lo > 4e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (sturm(a, b, k, mid) >= 1) hi = mid; else lo = mid;
  }
  *lam = 0.5 * (lo + hi);
  // inverse iteration on (T − σI), σ just below λ: tridiagonal LU with partial pivoting
  double* x = s;
  double* dl = wk;
  double* d = wk + k;
  double* du = wk + 2 * k;
  double* du2 = wk + 3 * k;
  for (int i = 0; i < k; ++i) x[i] = 1.0 + 0.01 * sin(1.0 + i);
  const double shift = *lam - 1e-14 * span;
  for (int itr = 0; itr < 3; ++itr) {
    for (int i = 0; i < k; ++i) d[i] = a[i] - shift;
    for (int i = 0; i < k - 1; ++i) dl[i] = du[i] = b[i];
    for (int i = 0; i < k; ++i) du2[i] = 0.0;
    for (int i = 0; i < k - 1; ++i) {
      if (fabs(d[i]) >= fabs(dl[i])) {
        if (d[i] == 0.0) d[i] = 1e-300;
        const double f = dl[i] / d[i];
        d[i + 1] -= f * du[i];
        x[i + 1] -= f * x[i];
        dl[i] = 0.0;
      } else {
        const double f = d[i] / dl[i];
        d[i] = dl[i];
        const double t = d[i + 1];
        d[i + 1] = du[i] - f * t;
        if (i < k - 2) {
          du2[i] = du[i + 1];
          du[i + 1] = -f * du2[i];
        }
        du[i] = t;
        const double tx = x[i];
        x[i] = x[i + 1];
        x[i + 1] = tx - f * x[i + 1];
      }
    }
    if (d[k - 1] == 0.0) d[k - 1] = 1e-300;
    x[k - 1] /= d[k - 1];
    if (k > 1) x[k - 2] = (x[k - 2] - du[k - 2] * x[k - 1]) / d[k - 2];
    for (int i = k - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) / d[i];
    double nrm = 0.0;
    for (int i = 0; i < k; ++i) nrm += x[i] * x[i];
    nrm = sqrt(nrm);
    for (int i = 0; i < k; ++i) x[i] /= nrm;
  }
}

__device__ double splitmix_u(uint64_t seed, int64_t j) {
  uint64_t z = seed + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

// Lanczos on Z = Q − blkdiag(Λ) with full re-orthogonalisation (O6, C19): λ_min,
// v in s.w (normalised, largest-|·| component positive); returns steps
__device__ int blanczos(const Sm& s, const BatchArgs& a, double tol, double* lam_out) {
  const int n = a.n, kmax = min(a.lanczos_max, n);
  double* V = s.V;
  for (int x = threadIdx.x; x < n; x += kBT) V[x] = splitmix_u(a.seed, x);
  __syncthreads();
  double nr = sqrt(bdot(V, V, n, s.red));
  for (int x = threadIdx.x; x < n; x += kBT) V[x] /= nr;
  __syncthreads();
  int k = 0;
  double lam = 0.0;
  for (k = 1; k <= kmax; ++k) {
    const double* vk = V + (k - 1) * n;
    for (int row = threadIdx.x; row < n; row += kBT) {  // w = Q v − Λ v
      double sum = 0.0;
      for (int q = 0; q < n; ++q) sum = fma(s.Q[row * n + q], vk[q], sum);
      const int i = row / 3, ra = row % 3;
      double l = 0.0;
      for (int b = 0; b < 3; ++b) l = fma(lam_at(s.LAM + 6 * i, ra, b), vk[3 * i + b], l);
      s.w[row] = sum - l;
    }
    __syncthreads();
    const double al = bdot(vk, s.w, n, s.red);
    if (threadIdx.x == 0) s.al[k - 1] = al;
    for (int pass = 0; pass < 2; ++pass) {  // classical GS against v_0..v_{k−1}, twice
      for (int j = threadIdx.x; j < k; j += kBT) {
        double c = 0.0;
        for (int x = 0; x < n; ++x) c = fma(V[j * n + x], s.w[x], c);
        s.TMP[j] = c;
      }
      __syncthreads();
      for (int x = threadIdx.x; x < n; x += kBT) {
        double sub = 0.0;
        for (int j = 0; j < k; ++j) sub = fma(V[j * n + x], s.TMP[j], sub);
        s.w[x] -= sub;
      }
      __syncthreads();
    }
    const double bk = sqrt(bdot(s.w, s.w, n, s.red));
    if (threadIdx.x == 0) {
      tri_min(s.al, s.be, k, &s.scal[0], s.sv, s.DD);
      const double res = fabs(bk * s.sv[k - 1]);
      s.scal[1] = (res <= tol || bk <= 1e-300 || k == n) ? 1.0 : 0.0;
      if (s.scal[1] == 0.0) s.be[k - 1] = bk;
    }
    __syncthreads();
    lam = s.scal[0];
    if (s.scal[1] != 0.0 || k == kmax) break;
    for (int x = threadIdx.x; x < n; x += kBT) V[k * n + x] = s.w[x] / bk;
    __syncthreads();
  }
  const int kk = min(k, kmax);
  for (int x = threadIdx.x; x < n; x += kBT) {  // Ritz vector
    double v = 0.0;
    for (int j = 0; j < kk; ++j) v = fma(V[j * n + x], s.sv[j], v);
    s.w[x] = v;
  }
  __syncthreads();
  const double vn = sqrt(bdot(s.w, s.w, n, s.red));
  if (threadIdx.x == 0) {  // sign: largest |·| component positive (first index on ties)
    int best = 0;
    for (int x = 1; x < n; ++x)
      if (fabs(s.w[x]) > fabs(s.w[best])) best = x;
    s.scal[2] = (s.w[best] < 0.0 ? -1.0 : 1.0) / vn;
  }
  __syncthreads();
  const double sg = s.scal[2];
  for (int x = threadIdx.x; x < n; x += kBT) s.w[x] *= sg;
  __syncthreads();
  *lam_out = lam;
  return kk;
}

// one tCG solve (O5): ETA, HETA; returns stop (1 negcurv, 2 exceeded, 3 converged, 4 maxinner)
__device__ int btcg(const Sm& s, const BatchArgs& a, double Delta, int* nh, int rc) {
  const int n = a.n, len = n * kBR;
  for (int e = threadIdx.x; e < len; e += kBT) {
    s.ETA[e] = 0.0;
    s.HETA[e] = 0.0;
    s.RR[e] = s.G[e];
    s.DEL[e] = -s.G[e];
  }
  __syncthreads();
  double z = bdot(s.RR, s.RR, len, s.red);
  const double r0 = sqrt(z);
  double e_Pe = 0.0, e_Pd = 0.0, d_Pd = z;
  int stop = 4;
  for (int j = 0; j < a.max_inner; ++j) {
    bhess(s, s.DEL, s.HDEL, n, a.N, rc);
    ++*nh;
    const double dHd = bdot(s.DEL, s.HDEL, len, s.red);
    const double alpha = dHd != 0.0 ? z / dHd : INFINITY;
    const double e_new = e_Pe + 2.0 * alpha * e_Pd + alpha * alpha * d_Pd;
    if (dHd <= 0.0 || e_new >= Delta * Delta) {
      const double tau = (-e_Pd + sqrt(e_Pd * e_Pd + d_Pd * (Delta * Delta - e_Pe))) / d_Pd;
      for (int e = threadIdx.x; e < len; e += kBT) {
        s.ETA[e] = fma(tau, s.DEL[e], s.ETA[e]);
        s.HETA[e] = fma(tau, s.HDEL[e], s.HETA[e]);
      }
      __syncthreads();
      stop = dHd <= 0.0 ? 1 : 2;
      break;
    }
    for (int e = threadIdx.x; e < len; e += kBT) {
      s.ETA[e] = fma(alpha, s.DEL[e], s.ETA[e]);
      s.HETA[e] = fma(alpha, s.HDEL[e], s.HETA[e]);
      s.RR[e] = fma(alpha, s.HDEL[e], s.RR[e]);
    }
    __syncthreads();
    e_Pe = e_new;
    bproject(s.Y, s.RR, a.N);
    const double z_old = z;
    z = bdot(s.RR, s.RR, len, s.red);
    if (sqrt(z) <= r0 * fmin(pow(r0, a.theta), a.kappa)) {
      stop = 3;
      break;
    }
    const double beta = z / z_old;
    for (int e = threadIdx.x; e < len; e += kBT) s.DEL[e] = fma(beta, s.DEL[e], -s.RR[e]);
    __syncthreads();
    e_Pd = beta * (e_Pd + alpha * d_Pd);
    d_Pd = z + beta * beta * d_Pd;
  }
  return stop;
}

// GM = false: Q, the 12 vectors and the Lanczos basis in shared memory (n ≤ 72).
// GM = true (n > 72, e.g. Thm 3's BAL-93 trials, n = 279): Q is read from
// global memory (L2-resident: one shared Q serves every trial), the vectors and
// the basis live in a per-instance global scratch (L1 / L2); only the reduction
// buffer stays in shared memory.  Same arithmetic, same order.
template <bool GM>
__global__ void __launch_bounds__(kBT, 1) k_batch_staircase(BatchArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int n = a.n, N = a.N, len = n * kBR;
  const int inst = blockIdx.x;
  const double* Qg = a.Q + (int64_t)inst * a.qstride;
  Sm s;
  double* p = GM ? a.scratch + (int64_t)inst * a.scratch_stride : smem;
  if (GM) {
    s.Q = const_cast<double*>(Qg);
  } else {
    s.Q = p;
    p += n * n;
  }
  double** vecs[12] = {&s.Y, &s.QY, &s.G, &s.ETA, &s.HETA, &s.RR, &s.DEL, &s.HDEL, &s.TMP, &s.YN, &s.DD, &s.QD};
  for (int q = 0; q < 12; ++q) {
    *vecs[q] = p;
    p += len;
  }
  s.LAM = p; p += 6 * N;
  s.V = p; p += (int64_t)min(a.lanczos_max, n) * n;
  s.w = p; p += n;
  s.al = p; p += n;
  s.be = p; p += n;
  s.sv = p; p += n;
  if (GM) p = smem;
  s.red = p; p += kBT;
  s.scal = p; p += 8;

  if (!GM)
    for (int e = threadIdx.x; e < n * n; e += kBT) s.Q[e] = Qg[e];
  for (int e = threadIdx.x; e < len; e += kBT) {
    const int row = e / kBR, c = e % kBR;
    s.Y[e] = (c < a.r0) ? a.Y0[((int64_t)inst * n + row) * a.r0 + c] : 0.0;
  }
  __syncthreads();
  double q2 = 0.0;
  for (int e = threadIdx.x; e < n * n; e += kBT) q2 = fma(s.Q[e], s.Q[e], q2);
  const double normQ = sqrt(bsum(q2, s.red));
  const double sc = fmax(1.0, normQ);
  const double tol = a.grad_tol * sc;
  int r = a.r0, hvps = 0, outer_tot = 0, lz_tot = 0, status = 0, certified = 0, converged = 0;
  double f = 0.0, gn = 0.0, lam_min = 0.0;
  const double eps = 2.220446049250313e-16;
  for (;;) {
    // ---------------------------------------------------------------- RTR (O4)
    const double Delta0 = a.delta0_coef * sqrt(3.0 * N), Dbar = a.delta_max_mult * Delta0;
    double Delta = Delta0;
    bmatvec(s.Q, n, s.Y, s.QY, r);
    bmult(s.Y, s.QY, s.LAM, N);
    bsublam(s.QY, s.LAM, s.Y, 2.0, 2.0, s.G, n);
    f = bdot(s.Y, s.QY, len, s.red);
    int accepts = 0, it = 0;
    converged = 0;
    for (it = 0; it <= a.max_outer; ++it) {
      gn = sqrt(bdot(s.G, s.G, len, s.red));
      if (gn <= tol) {
        converged = 1;
        break;
      }
      if (it == a.max_outer) break;
      const int stop = btcg(s, a, Delta, &hvps, r);
      if (bretract(s.Y, s.ETA, 1.0, a.c_floor, s.YN, s.DD, N, s.red)) {
        status = XM_ERETRACT;
        break;
      }
      bmatvec(s.Q, n, s.DD, s.QD, r);
      const double df = 2.0 * bdot(s.QY, s.DD, len, s.red) + bdot(s.DD, s.QD, len, s.red);
      const double mdec = -bdot(s.G, s.ETA, len, s.red) - 0.5 * bdot(s.ETA, s.HETA, len, s.red);
      const double reg = fmax(1.0, fabs(f)) * eps * 1e3;
      const double rho = (-df + reg) / (mdec + reg);
      if (!(rho >= 0.25) || isnan(rho)) Delta /= 4.0;
      else if (rho > 0.75 && (stop == 1 || stop == 2)) Delta = fmin(2.0 * Delta, Dbar);
      if (rho > a.rho_prime) {
        ++accepts;
        for (int e = threadIdx.x; e < len; e += kBT) s.Y[e] = s.YN[e];
        __syncthreads();
        if (a.refresh_every > 0 && accepts % a.refresh_every == 0) {
          bmatvec(s.Q, n, s.Y, s.QY, r);
        } else {
          for (int e = threadIdx.x; e < len; e += kBT) s.QY[e] += s.QD[e];
          __syncthreads();
        }
        f = bdot(s.Y, s.QY, len, s.red);
        bmult(s.Y, s.QY, s.LAM, N);
        bsublam(s.QY, s.LAM, s.Y, 2.0, 2.0, s.G, n);
      }
    }
    outer_tot += it;
    if (status) break;
    // fresh QY, Λ, gradient before the certificate
    bmatvec(s.Q, n, s.Y, s.QY, r);
    bmult(s.Y, s.QY, s.LAM, N);
    bsublam(s.QY, s.LAM, s.Y, 2.0, 2.0, s.G, n);
    f = bdot(s.Y, s.QY, len, s.red);
    gn = sqrt(bdot(s.G, s.G, len, s.red));
    // ------------------------------------------------------------ certificate (O6)
    lz_tot += blanczos(s, a, a.eig_tol * sc, &lam_min);
    const bool ok = lam_min >= -a.cert_tol * sc;
    certified = (ok && converged) ? 1 : 0;
    if (ok || !converged || r >= a.rcap) {
      if (!converged) status = XM_NOT_CONVERGED;
      else if (!ok) status = XM_UNCERTIFIED;
      break;
    }
    // ------------------------------------------------------------ escape (O7, C9)
    for (int e = threadIdx.x; e < len; e += kBT) {
      const int row = e / kBR, c = e % kBR;
      s.ETA[e] = (c == r) ? s.w[row] : 0.0;  // direction [0, v]
    }
    __syncthreads();
    double alpha = 1.0;
    int done = 0;
    for (int h = 0; h <= 60; ++h) {
      bretract(s.Y, s.ETA, alpha, a.c_floor, s.YN, s.DD, N, s.red);
      bmatvec(s.Q, n, s.DD, s.QD, r + 1);  // the escape fills column r
      const double df = 2.0 * bdot(s.QY, s.DD, len, s.red) + bdot(s.DD, s.QD, len, s.red);
      if (df < 0.0) {
        for (int e = threadIdx.x; e < len; e += kBT) s.Y[e] = s.YN[e];
        __syncthreads();
        done = 1;
        break;
      }
      alpha *= 0.5;
    }
    if (!done) {
      status = XM_EESCAPE;
      break;
    }
    ++r;
  }
  double* Yo = a.Yout + (int64_t)inst * len;
  for (int e = threadIdx.x; e < len; e += kBT) Yo[e] = s.Y[e];
  if (threadIdx.x == 0) {
    xm_batch_result& o = a.res[inst];
    o.f = f;
    o.grad_norm = gn;
    o.lambda_min = lam_min;
    o.normQ = normQ;
    o.r = r;
    o.certified = certified;
    o.status = status;
    o.hvps = hvps;
    o.outer_iters = outer_tot;
    o.lanczos_steps = lz_tot;
  }
}
}  // namespace

// doubles of one instance's vectors, multipliers and Lanczos basis
static size_t batch_vec_doubles(int N, int lanczos_max) {
  const int n = 3 * N;
  return 12 * (size_t)n * kBR + 6 * (size_t)N + (size_t)std::min(lanczos_max, n) * n + 4 * (size_t)n;
}
size_t batch_smem_bytes(int N, int lanczos_max) {
  const int n = 3 * N;
  if (N > kBNmax) return sizeof(double) * (kBT + 8);  // GM layout
  return sizeof(double) * ((size_t)n * n + batch_vec_doubles(N, lanczos_max) + kBT + 8);
}

void batch_staircase(xm_ctx* c, int B, int N, const double* Q_dev, int64_t qstride,
                     const double* Y0_dev, int r0, double* Yout_dev, xm_batch_result* res_dev) {
  if (N < 1 || N > kBNmaxGM)
    throw Error(XM_EINVAL, "batched solve: 1 ≤ N ≤ 400 frames per instance");
  const int rcap = std::min(c->opt.rank_cap, kBR);
  if (r0 < 3 || r0 > rcap) throw Error(XM_EINVAL, "batched solve: 3 ≤ r0 ≤ min(rank_cap, 8)");
  BatchArgs a{};
  a.B = B;
  a.N = N;
  a.n = 3 * N;
  a.r0 = r0;
  a.rcap = rcap;
  a.Q = Q_dev;
  a.qstride = qstride;
  a.Y0 = Y0_dev;
  a.Yout = Yout_dev;
  a.res = res_dev;
  const xm_options& o = c->opt;
  a.grad_tol = o.grad_tol;
  a.delta0_coef = o.delta0_coef;
  a.delta_max_mult = o.delta_max_mult;
  a.rho_prime = o.rho_prime;
  a.kappa = o.tcg_kappa;
  a.theta = o.tcg_theta;
  a.eig_tol = o.eig_tol;
  a.cert_tol = o.cert_tol;
  a.c_floor = o.scale_floor;
  a.max_inner = o.tcg_max_inner;
  a.max_outer = o.max_outer;
  a.refresh_every = o.refresh_every;
  a.lanczos_max = o.lanczos_max;
  a.seed = o.seed;
  const size_t smem = batch_smem_bytes(N, a.lanczos_max);
  if (N <= kBNmax) {
    ensure_smem_attr((const void*)k_batch_staircase<false>, smem);
    k_batch_staircase<false><<<B, kBT, smem, c->stream>>>(a);
  } else {
    a.scratch_stride = (int64_t)round_up((int64_t)batch_vec_doubles(N, a.lanczos_max), 32);
    DBuf<double>& sc = scratch_f64(c, "batch_scratch");
    sc.alloc((size_t)B * a.scratch_stride);
    a.scratch = sc.p;
    k_batch_staircase<true><<<B, kBT, smem, c->stream>>>(a);
  }
  XM_CHECK_LAUNCH();
  count_launch(c);
}

}  // namespace xm
