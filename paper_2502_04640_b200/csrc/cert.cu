// cert.cu — H11 certificate (Lanczos λ_min of Z = Q − blkdiag(Λ)) and
// H13 rounding + recovery.
//
//  * Lanczos with full re-orthogonalisation (two classical Gram–Schmidt passes,
//    S:377-385, reading C19); every O(n) operation runs on the device, the
//    host only keeps the k scalars (α_j, β_j) of the tridiagonal T_k and
//    extracts its smallest Ritz pair (Sturm bisection + inverse iteration).
//  * Rounding: Gram YᵀY (r×r) → top-3 eigenvectors W₃ (host Jacobi on
//    r ≤ 12) → Y₃ = Y W₃ → per camera: gauge fix by the polar factor of block 0
//    (Eq. (12)), s_i = ‖B_i‖_F/√3, nearest SO(3) (det < 0 ⇒ flip, Eq. (9)).
//  * Recovery (Eq. (4)): T = −K̄⁻¹ C̄ Y₃ = −L⁻ᵀ (G Y₃), t_0 = 0;
//    p_k = Σ_{e∈k} w_e (Ū_i ũ_e + t_i) / W_k.
#include "xm_internal.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace xm {

// ------------------------------------------------------------------ start vector
// splitmix64 counter stream, identical to synth.scenes.splitmix64_uniform
__global__ void k_splitmix(int64_t n, uint64_t seed, double* __restrict__ out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint64_t z = seed + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  out[j] = 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

void splitmix_uniform(xm_ctx* c, int64_t n, uint64_t seed, double* out) {
  k_splitmix<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, seed, out);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

// x ← x / sqrt(*sumsq);  optionally record sqrt into beta_out
__global__ void k_normalize(int64_t n, const double* __restrict__ sumsq, const double* __restrict__ x,
                            double* __restrict__ out, double* __restrict__ beta_out) {
  double nrm = sqrt(*sumsq);
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t == 0 && beta_out) *beta_out = nrm;
  if (t >= n) return;
  out[t] = (nrm > 0.0) ? x[t] / nrm : 0.0;
}

// c[j] = ⟨V_j, w⟩ for j < k  (one block per basis vector, fixed tree)
__global__ void __launch_bounds__(256) k_gemv_t(const double* __restrict__ V, int64_t ldv, int64_t n,
                                                const double* __restrict__ w,
                                                double* __restrict__ c) {
  __shared__ double sh[256];
  const double* row = V + (int64_t)blockIdx.x * ldv;
  double acc = 0.0;
  for (int64_t x = threadIdx.x; x < n; x += 256) acc = fma(row[x], w[x], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) c[blockIdx.x] = sh[0];
}

// part[chunk][x] = Σ_{j in chunk} V_j[x]·c[j]  (chunks of 64 basis vectors)
constexpr int kGemvChunk = 64;
__global__ void __launch_bounds__(256) k_gemv_n_part(const double* __restrict__ V, int64_t ldv,
                                                     int64_t n, int k, const double* __restrict__ c,
                                                     double* __restrict__ part) {
  int64_t x = blockIdx.x * 256 + threadIdx.x;
  int j0 = blockIdx.y * kGemvChunk;
  int j1 = min(k, j0 + kGemvChunk);
  if (x >= n) return;
  double acc = 0.0;
  for (int j = j0; j < j1; ++j) acc = fma(V[(int64_t)j * ldv + x], c[j], acc);
  part[(int64_t)blockIdx.y * n + x] = acc;
}
// w[x] = sign·w[x] + scale·Σ_chunk part[chunk][x]
__global__ void k_gemv_n_fin(int64_t n, int nchunk, const double* __restrict__ part, double scale,
                             double keep, double* __restrict__ w) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  double s = 0.0;
  for (int q = 0; q < nchunk; ++q) s += part[(int64_t)q * n + x];
  w[x] = keep * w[x] + scale * s;
}

// argmax |x| (first index on ties), one block
__global__ void k_argmax_abs(int64_t n, const double* __restrict__ x, double* __restrict__ out) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  double best = -1.0;
  int64_t bi = 0;
  for (int64_t t = threadIdx.x; t < n; t += 256) {
    double a = fabs(x[t]);
    if (a > best) { best = a; bi = t; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      double a = sv[threadIdx.x + s];
      int64_t ia = si[threadIdx.x + s];
      if (a > sv[threadIdx.x] || (a == sv[threadIdx.x] && ia < si[threadIdx.x])) {
        sv[threadIdx.x] = a;
        si[threadIdx.x] = ia;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = (x[si[0]] < 0.0) ? -1.0 : 1.0;
}
__global__ void k_scale_by(int64_t n, const double* __restrict__ sgn, double* __restrict__ x) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) x[t] *= *sgn;
}

// ------------------------------------------------------------------ host tridiagonal
// Smallest eigenpair of the symmetric tridiagonal T (diag a[0..k), off b[0..k-1)).
static int sturm_count(const std::vector<double>& a, const std::vector<double>& b, int k,
                       double x) {
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

// tridiagonal solve (T − λI) x = rhs with partial pivoting (gtsv-style)
static void gtsv(int k, std::vector<double> dl, std::vector<double> d, std::vector<double> du,
                 std::vector<double>& x) {
  std::vector<double> du2(k, 0.0);
  for (int i = 0; i < k - 1; ++i) {
    if (std::fabs(d[i]) >= std::fabs(dl[i])) {
      if (d[i] == 0.0) d[i] = 1e-300;
      double f = dl[i] / d[i];
      d[i + 1] -= f * du[i];
      x[i + 1] -= f * x[i];
      dl[i] = 0.0;
    } else {
      double f = d[i] / dl[i];
      d[i] = dl[i];
      double t = d[i + 1];
      d[i + 1] = du[i] - f * t;
      if (i < k - 2) {
        du2[i] = du[i + 1];
        du[i + 1] = -f * du2[i];
      }
      du[i] = t;
      std::swap(x[i], x[i + 1]);
      x[i + 1] -= f * x[i];
    }
  }
  if (d[k - 1] == 0.0) d[k - 1] = 1e-300;
  x[k - 1] /= d[k - 1];
  if (k > 1) x[k - 2] = (x[k - 2] - du[k - 2] * x[k - 1]) / d[k - 2];
  for (int i = k - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) / d[i];
}

static void tridiag_min(const std::vector<double>& a, const std::vector<double>& b, int k,
                        double& lam, std::vector<double>& s) {
  s.assign(k, 0.0);
  if (k == 1) {
    lam = a[0];
    s[0] = 1.0;
    return;
  }
  double lo = a[0], hi = a[0];
  for (int i = 0; i < k; ++i) {
    double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i < k - 1 ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  double span = std::max(hi - lo, 1e-300);
  for (int it = 0; it < 200 && hi - lo > 4e-16 * std::max(std::fabs(lo), std::fabs(hi)) + 1e-300;
       ++it) {
    double mid = 0.5 * (lo + hi);
    if (sturm_count(a, b, k, mid) >= 1) hi = mid; else lo = mid;
  }
  lam = 0.5 * (lo + hi);
  // inverse iteration
  std::vector<double> x(k, 1.0);
  for (int i = 0; i < k; ++i) x[i] = 1.0 + 0.01 * std::sin(1.0 + i);
  double shift = lam - 1e-14 * span;
  for (int it = 0; it < 3; ++it) {
    std::vector<double> d(k), dl(k - 1), du(k - 1);
    for (int i = 0; i < k; ++i) d[i] = a[i] - shift;
    for (int i = 0; i < k - 1; ++i) dl[i] = du[i] = b[i];
    gtsv(k, dl, d, du, x);
    double nrm = 0.0;
    for (double v : x) nrm += v * v;
    nrm = std::sqrt(nrm);
    for (double& v : x) v /= nrm;
  }
  s = x;
}

// y = X v for a lower-triangular X (row-major, ld): one block per row, x ≤ row
__global__ void __launch_bounds__(256) k_trmv_lower(const double* __restrict__ X, int64_t ldx,
                                                    int64_t n, const double* __restrict__ v,
                                                    double* __restrict__ y) {
  __shared__ double sh[256];
  const int64_t row = blockIdx.x;
  const double* xr = X + row * ldx;
  double acc = 0.0;
  for (int64_t x = threadIdx.x; x <= row; x += 256) acc = fma(xr[x], v[x], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) y[row] = sh[0];
}

// Lanczos (full re-orthogonalisation) for the smallest eigenpair of
//   op.X == nullptr : Z = Q − blkdiag(Λ)               (Alg. 1 l.9-12, C19)
//   op.X != nullptr : −Xᵀ X  with X = L⁻¹, LLᵀ = Z + sI  (shift-invert: its
//                     smallest Ritz value is −1/(λ_min(Z) + s))
bool lanczos(xm_ctx* c, double tol_abs, int max_steps, double* lambda, int* steps,
             double* vec_dev, const LanczosOp& op) {
  const int64_t n = c->n;
  const int kmax = (int)std::max<int64_t>(1, std::min<int64_t>(max_steps, n));
  const int64_t ldv = round_up(n, 32);
  c->lz_V.alloc((size_t)(kmax + 1) * ldv);
  c->lz_w.alloc(round_up(n, 32) * std::max(1, c->world) + 64);
  c->lz_c.alloc((size_t)2 * (kmax + 1) + 64);
  int nchunk_max = ceil_div(kmax + 1, kGemvChunk);
  if (op.X) nchunk_max = std::max(nchunk_max, ceil_div(n, kGemvChunk));
  c->lz_part.alloc((size_t)nchunk_max * n + 4096);
  c->tmp.alloc((size_t)c->n_alloc * 4);
  double* alphas = c->lz_c.p;                    // device α_j
  double* betas = c->lz_c.p + (kmax + 1);        // device β_j
  DBuf<double>& cbuf = scratch_f64(c, "lz_cbuf");
  cbuf.alloc(kmax + 64);
  double* dots = c->lz_part.p + (size_t)nchunk_max * n;  // kDotBlocks partials
  double* scal = c->scal.p + 48;

  // v_0 = normalised splitmix64 stream
  k_splitmix<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, c->opt.seed, c->lz_w.p);
  dot_flat(c, c->lz_w.p, c->lz_w.p, n, dots, kDotBlocks);
  reduce_partials(c, dots, kDotBlocks, 1, scal);
  k_normalize<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, scal, c->lz_w.p, c->lz_V.p, nullptr);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);

  std::vector<double> ha, hb, s;
  double lam = 0.0;
  int k = 0;
  bool converged = false;
  const int check_every = 8;
  bool done = false;
  while (!done) {
    int batch_end = std::min(kmax, k + check_every);
    for (; k < batch_end; ++k) {
      const double* vk = c->lz_V.p + (int64_t)k * ldv;
      // w = Z v_k = Q v_k − Λ v_k   (or −Xᵀ X v_k)
      if (op.X) {
        double* y = c->tmp.p;
        k_trmv_lower<<<(unsigned)n, 256, 0, c->stream>>>(op.X, op.ldx, n, vk, y);
        const int nch = ceil_div(n, kGemvChunk);
        k_gemv_n_part<<<dim3(ceil_div(n, 256), nch), 256, 0, c->stream>>>(op.X, op.ldx, n, (int)n, y,
                                                                         c->lz_part.p);
        k_gemv_n_fin<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, nch, c->lz_part.p, -1.0, 0.0,
                                                            c->lz_w.p);
        XM_CHECK_LAUNCH();
        count_launch(c, 3);
        dot_flat(c, vk, c->lz_w.p, n, dots, kDotBlocks);
        reduce_partials(c, dots, kDotBlocks, 1, alphas + k);
      } else if (fused_epilogues(c)) {
        SpmmEpiArgs ep{};
        ep.out = c->lz_w.p;
        ep.lam = c->lam.p;
        ep.partials = dots;
        spmm(c, vk, 1, EPI_ZMUL, ep);  // w = Qv − Λv, partials of ⟨v, w⟩
        reduce_partials(c, dots, spmm_grid(c, 1), 1, alphas + k);
      } else {
        spmm_full(c, vk, 1, c->tmp.p, nullptr);
        zmul(c, vk, c->tmp.p, c->lz_w.p);
        dot_flat(c, vk, c->lz_w.p, n, dots, kDotBlocks);
        reduce_partials(c, dots, kDotBlocks, 1, alphas + k);
      }
      // full re-orthogonalisation against v_0..v_k, two passes
      for (int pass = 0; pass < 2; ++pass) {
        k_gemv_t<<<k + 1, 256, 0, c->stream>>>(c->lz_V.p, ldv, n, c->lz_w.p, cbuf.p);
        int nch = ceil_div(k + 1, kGemvChunk);
        k_gemv_n_part<<<dim3(ceil_div(n, 256), nch), 256, 0, c->stream>>>(c->lz_V.p, ldv, n, k + 1,
                                                                         cbuf.p, c->lz_part.p);
        k_gemv_n_fin<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, nch, c->lz_part.p, -1.0, 1.0,
                                                            c->lz_w.p);
        XM_CHECK_LAUNCH();
        count_launch(c, 3);
      }
      dot_flat(c, c->lz_w.p, c->lz_w.p, n, dots, kDotBlocks);
      reduce_partials(c, dots, kDotBlocks, 1, scal);
      k_normalize<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, scal, c->lz_w.p,
                                                          c->lz_V.p + (int64_t)(k + 1) * ldv,
                                                          betas + k);
      XM_CHECK_LAUNCH();
      count_launch(c);
    }
    int kk = k;  // number of Lanczos vectors processed
    ha.resize(kk);
    hb.resize(kk);
    XM_CUDA(cudaMemcpyAsync(ha.data(), alphas, kk * 8, cudaMemcpyDeviceToHost, c->stream));
    XM_CUDA(cudaMemcpyAsync(hb.data(), betas, kk * 8, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    tridiag_min(ha, hb, kk, lam, s);
    double res = std::fabs(hb[kk - 1] * s[kk - 1]);
    // shift-invert: θ = −1/(λ + s) ⇒ |dλ| = |dθ|/θ², so the Z-tolerance maps to tol·θ²
    const double tol_k = op.X ? tol_abs * lam * lam : tol_abs;
    const double scale_k = op.X ? std::fabs(lam) : std::max(1.0, c->normQ);
    bool breakdown = hb[kk - 1] <= 1e-14 * scale_k;
    converged = res <= tol_k || breakdown || kk >= (int)n;
    if (converged || kk >= kmax) done = true;
  }
  *lambda = lam;
  *steps = k;
  if (vec_dev) {
    // Ritz vector x = Σ_j s_j v_j, normalised, largest-|·| component positive
    XM_CUDA(cudaMemcpyAsync(cbuf.p, s.data(), k * 8, cudaMemcpyHostToDevice, c->stream));
    int nch = ceil_div(k, kGemvChunk);
    k_gemv_n_part<<<dim3(ceil_div(n, 256), nch), 256, 0, c->stream>>>(c->lz_V.p, ldv, n, k, cbuf.p,
                                                                     c->lz_part.p);
    k_gemv_n_fin<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, nch, c->lz_part.p, 1.0, 0.0, vec_dev);
    XM_CHECK_LAUNCH();
    dot_flat(c, vec_dev, vec_dev, n, dots, kDotBlocks);
    reduce_partials(c, dots, kDotBlocks, 1, scal);
    k_normalize<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, scal, vec_dev, vec_dev, nullptr);
    k_argmax_abs<<<1, 256, 0, c->stream>>>(n, vec_dev, scal + 1);
    k_scale_by<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, scal + 1, vec_dev);
    XM_CHECK_LAUNCH();
    count_launch(c, 5);
    sync(c);
  }
  return converged;
}

// ================================================================== rounding
// Gram entries G[p][q] = Σ_x Y[x][p] Y[x][q], one block per (p, q ≥ p)
__global__ void __launch_bounds__(256) k_gram(int64_t n, int r, const double* __restrict__ Y,
                                              double* __restrict__ out) {
  __shared__ double sh[256];
  int pair = blockIdx.x, p = 0;
  int rem = pair;
  while (rem >= r - p) { rem -= r - p; ++p; }
  int q = p + rem;
  double acc = 0.0;
  for (int64_t x = threadIdx.x; x < n; x += 256) acc = fma(Y[x * r + p], Y[x * r + q], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[p * r + q] = sh[0];
    out[q * r + p] = sh[0];
  }
}

// Y3 = Y W3  (W3: r × 3, row-major)
__global__ void k_y_times_w3(int64_t n, int r, const double* __restrict__ Y,
                             const double* __restrict__ W3, double* __restrict__ Y3) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  double a0 = 0, a1 = 0, a2 = 0;
  for (int p = 0; p < r; ++p) {
    double y = Y[x * r + p];
    a0 = fma(y, W3[p * 3 + 0], a0);
    a1 = fma(y, W3[p * 3 + 1], a1);
    a2 = fma(y, W3[p * 3 + 2], a2);
  }
  Y3[x * 3] = a0;
  Y3[x * 3 + 1] = a1;
  Y3[x * 3 + 2] = a2;
}

// 3×3 symmetric Jacobi eigen-decomposition (ascending eigenvalues, V columns)
__host__ __device__ inline void jacobi3(double A[3][3], double V[3][3], double ev[3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    double dn = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
    if (off <= 1e-34 * dn || off == 0.0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 3; ++k) {
          double akp = A[k][p], akq = A[k][q];
          A[k][p] = cs * akp - sn * akq;
          A[k][q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = A[p][k], aqk = A[q][k];
          A[p][k] = cs * apk - sn * aqk;
          A[q][k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = cs * vkp - sn * vkq;
          V[k][q] = sn * vkp + cs * vkq;
        }
      }
  }
  ev[0] = A[0][0];
  ev[1] = A[1][1];
  ev[2] = A[2][2];
  // sort ascending (columns of V along)
  for (int i = 0; i < 2; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (ev[j] < ev[i]) {
        double t = ev[i]; ev[i] = ev[j]; ev[j] = t;
        for (int k = 0; k < 3; ++k) { double u = V[k][i]; V[k][i] = V[k][j]; V[k][j] = u; }
      }
}

// Orthogonal polar factor of B (3×3) and the nearest SO(3) matrix.
//   B = U Σ Vᵀ (σ₁ ≥ σ₂ ≥ σ₃): u₁ = Bv₁/σ₁, u₂ = Bv₂/σ₂ (orthogonalised),
//   u₃ = ±u₁×u₂.  polar = U Vᵀ (det = sign det B); so3 = [u₁,u₂,det(V)·u₁×u₂] Vᵀ.
__device__ inline bool polar3(const double B[3][3], double P[3][3], double Rso3[3][3],
                              double* detB) {
  double S[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += B[k][i] * B[k][j];
      S[i][j] = s;
    }
  double V[3][3], ev[3];
  jacobi3(S, V, ev);
  // descending order: columns 2, 1, 0
  double v1[3] = {V[0][2], V[1][2], V[2][2]}, v2[3] = {V[0][1], V[1][1], V[2][1]},
         v3[3] = {V[0][0], V[1][0], V[2][0]};
  double u1[3], u2[3];
  for (int i = 0; i < 3; ++i) {
    u1[i] = B[i][0] * v1[0] + B[i][1] * v1[1] + B[i][2] * v1[2];
    u2[i] = B[i][0] * v2[0] + B[i][1] * v2[1] + B[i][2] * v2[2];
  }
  double n1 = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
  if (!(n1 > 0)) return false;
  for (int i = 0; i < 3; ++i) u1[i] /= n1;
  double d = u1[0] * u2[0] + u1[1] * u2[1] + u1[2] * u2[2];
  for (int i = 0; i < 3; ++i) u2[i] -= d * u1[i];
  double n2 = sqrt(u2[0] * u2[0] + u2[1] * u2[1] + u2[2] * u2[2]);
  if (!(n2 > 0)) return false;
  for (int i = 0; i < 3; ++i) u2[i] /= n2;
  double u3[3] = {u1[1] * u2[2] - u1[2] * u2[1], u1[2] * u2[0] - u1[0] * u2[2],
                  u1[0] * u2[1] - u1[1] * u2[0]};
  double dB = B[0][0] * (B[1][1] * B[2][2] - B[1][2] * B[2][1]) -
              B[0][1] * (B[1][0] * B[2][2] - B[1][2] * B[2][0]) +
              B[0][2] * (B[1][0] * B[2][1] - B[1][1] * B[2][0]);
  double dV = v1[0] * (v2[1] * v3[2] - v2[2] * v3[1]) - v1[1] * (v2[0] * v3[2] - v2[2] * v3[0]) +
              v1[2] * (v2[0] * v3[1] - v2[1] * v3[0]);
  *detB = dB;
  double sgn_pol = (dB < 0 ? -1.0 : 1.0) * (dV < 0 ? -1.0 : 1.0);
  double sgn_so3 = (dV < 0 ? -1.0 : 1.0);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double common = u1[i] * v1[j] + u2[i] * v2[j];
      P[i][j] = common + sgn_pol * u3[i] * v3[j];
      Rso3[i][j] = common + sgn_so3 * u3[i] * v3[j];
    }
  return true;
}

// gauge: O₀ = polar(B₀), s₀ = ‖B₀‖/√3  (B_i = Y3_iᵀ)
__global__ void k_gauge0(const double* __restrict__ Y3, double* __restrict__ g, int* __restrict__ err) {
  double B[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) B[a][b] = Y3[b * 3 + a];  // Ū_0 = Y3_0ᵀ
  double fn = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) fn += B[a][b] * B[a][b];
  double s0 = sqrt(fn / 3.0);
  double P[3][3], Rs[3][3], dB;
  if (!(s0 > 1e-12) || !polar3(B, P, Rs, &dB)) {
    atomicOr(err, 2);
    s0 = 1.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) P[a][b] = (a == b);
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) g[a * 3 + b] = P[a][b];
  g[9] = s0;
}

__global__ void k_round_blocks(int N, const double* __restrict__ Y3, const double* __restrict__ g,
                               double* __restrict__ Rout, double* __restrict__ sout,
                               double* __restrict__ Yr, int* __restrict__ flips,
                               int* __restrict__ err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double O[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) O[a][b] = g[a * 3 + b];
  double s0 = g[9];
  double B[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      // (O₀ᵀ Ū_i)[a][b] / s₀,  Ū_i[k][b] = Y3[(3i+b)*3 + k]
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += O[k][a] * Y3[(3 * (int64_t)i + b) * 3 + k];
      B[a][b] = s / s0;
    }
  double fn = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) fn += B[a][b] * B[a][b];
  double si = sqrt(fn / 3.0);
  double R[3][3];
  if (i == 0) {
    si = 1.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) R[a][b] = (a == b);
  } else {
    double P[3][3], dB;
    if (!(si > 1e-12) || !polar3(B, P, R, &dB)) {
      atomicOr(err, 2);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) R[a][b] = (a == b);
    } else if (dB < 0.0) {
      atomicAdd(flips, 1);
    }
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      Rout[9 * (int64_t)i + 3 * a + b] = R[a][b];
      // Yr rows 3i+b: Y_i = Ū_iᵀ, Ū_i = s_i R_i  ⇒ Yr[3i+b][a] = s_i R[a][b]
      Yr[(3 * (int64_t)i + b) * 3 + a] = si * R[a][b];
    }
  sout[i] = si;
}

// rhs[j][c] = Σ_x G[j][x] Yr[x][c]  (warp per row of G)
__global__ void k_g_times_y3(int m, int64_t n, int64_t ldg, const double* __restrict__ G,
                             const double* __restrict__ Yr, double* __restrict__ rhs) {
  int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (j >= m) return;
  const double* row = G + (int64_t)j * ldg;
  double a0 = 0, a1 = 0, a2 = 0;
  for (int64_t x = lane; x < n; x += 32) {
    double gv = row[x];
    a0 = fma(gv, Yr[x * 3], a0);
    a1 = fma(gv, Yr[x * 3 + 1], a1);
    a2 = fma(gv, Yr[x * 3 + 2], a2);
  }
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (lane == 0) {
    rhs[j * 3] = a0;
    rhs[j * 3 + 1] = a1;
    rhs[j * 3 + 2] = a2;
  }
}

// Lᵀ x = rhs (3 right-hand sides), t_{j+1} = −x_j: blocked back substitution,
// one launch per 64-row block from the bottom.  Every CTA solves the block's
// 64 × 64 triangle redundantly from its (final) right-hand sides (smem), CTA 0
// writes x_b as t, and each CTA updates its slice of the rows above,
// rhs_l −= Σ_{j ∈ b} L_jl x_j (rows j of L: coalesced in l).
constexpr int kBS = 64;
__global__ void __launch_bounds__(256) k_backsub_block(int kb, int nb, int64_t ldl,
                                                       const double* __restrict__ L,
                                                       double* __restrict__ rhs,
                                                       double* __restrict__ t) {
  __shared__ double Ld[kBS][kBS + 1];
  __shared__ double xb[kBS][3];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    Ld[i][j] = (j <= i) ? L[(int64_t)(kb + i) * ldl + kb + j] : 0.0;
  }
  for (int e = threadIdx.x; e < nb * 3; e += blockDim.x) xb[e / 3][e % 3] = rhs[(int64_t)kb * 3 + e];
  __syncthreads();
  if (threadIdx.x < 3) {
    const int cc = threadIdx.x;
    for (int i = nb - 1; i >= 0; --i) {
      double v = xb[i][cc];
      for (int k = i + 1; k < nb; ++k) v = fma(-Ld[k][i], xb[k][cc], v);
      xb[i][cc] = v / Ld[i][i];
    }
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < nb * 3; e += blockDim.x) t[(int64_t)(kb + 1) * 3 + e] = -xb[e / 3][e % 3];
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= kb) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int i = 0; i < nb; ++i) {
    const double lv = L[(int64_t)(kb + i) * ldl + l];
    a0 = fma(lv, xb[i][0], a0);
    a1 = fma(lv, xb[i][1], a1);
    a2 = fma(lv, xb[i][2], a2);
  }
  rhs[(int64_t)l * 3] -= a0;
  rhs[(int64_t)l * 3 + 1] -= a1;
  rhs[(int64_t)l * 3 + 2] -= a2;
}

// p_k = Σ_{e ∈ track k} w_e (s_i R_i ũ_e + t_i) / W_k
__global__ void k_points(int M, const int32_t* __restrict__ off, const int32_t* __restrict__ e_fr,
                         const double* __restrict__ e_pts, const double* __restrict__ e_w,
                         const double* __restrict__ W, const double* __restrict__ R,
                         const double* __restrict__ s, const double* __restrict__ t,
                         double* __restrict__ p) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  if (!(W[k] > 0.0)) {
    p[3 * k] = p[3 * k + 1] = p[3 * k + 2] = nan("");
    return;
  }
  double acc[3] = {0, 0, 0};
  for (int e = off[k]; e < off[k + 1]; ++e) {
    int i = e_fr[e];
    const double* Ri = R + 9 * (int64_t)i;
    double u0 = e_pts[3 * e], u1 = e_pts[3 * e + 1], u2 = e_pts[3 * e + 2];
    for (int a = 0; a < 3; ++a) {
      double x = s[i] * (Ri[3 * a] * u0 + Ri[3 * a + 1] * u1 + Ri[3 * a + 2] * u2) + t[3 * i + a];
      acc[a] = fma(e_w[e], x, acc[a]);
    }
  }
  for (int a = 0; a < 3; ++a) p[3 * k + a] = acc[a] / W[k];
}

// r×r symmetric Jacobi (host), eigenvalues descending with vectors in columns
static void jacobi_host(int r, std::vector<double> A, std::vector<double>& V,
                        std::vector<double>& ev) {
  V.assign(r * r, 0.0);
  for (int i = 0; i < r; ++i) V[i * r + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, dn = 0.0;
    for (int p = 0; p < r; ++p)
      for (int q = 0; q < r; ++q) (p == q ? dn : off) += A[p * r + q] * A[p * r + q];
    if (off <= 1e-32 * dn || off == 0.0) break;
    for (int p = 0; p < r - 1; ++p)
      for (int q = p + 1; q < r; ++q) {
        double apq = A[p * r + q];
        if (apq == 0.0) continue;
        double theta = (A[q * r + q] - A[p * r + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < r; ++k) {
          double akp = A[k * r + p], akq = A[k * r + q];
          A[k * r + p] = cs * akp - sn * akq;
          A[k * r + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < r; ++k) {
          double apk = A[p * r + k], aqk = A[q * r + k];
          A[p * r + k] = cs * apk - sn * aqk;
          A[q * r + k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < r; ++k) {
          double vkp = V[k * r + p], vkq = V[k * r + q];
          V[k * r + p] = cs * vkp - sn * vkq;
          V[k * r + q] = sn * vkp + cs * vkq;
        }
      }
  }
  ev.resize(r);
  std::vector<int> idx(r);
  for (int i = 0; i < r; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return A[a * r + a] > A[b * r + b]; });
  std::vector<double> V2(r * r);
  for (int j = 0; j < r; ++j) {
    ev[j] = A[idx[j] * r + idx[j]];
    for (int k = 0; k < r; ++k) V2[k * r + j] = V[k * r + idx[j]];
  }
  V = V2;
}

void round_recover_device(xm_ctx* c) {
  const int r = c->r, N = c->N, M = c->M;
  const int64_t n = c->n;
  c->Yr.alloc((size_t)n * 3 + 64);
  c->Rs.alloc((size_t)N * 9);
  c->s_out.alloc(N);
  c->t_out.alloc((size_t)N * 3);
  c->p_out.alloc((size_t)M * 3);
  c->rhs.alloc((size_t)std::max(N, 1) * 3 + 64);
  DBuf<double>& gram = scratch_f64(c, "rnd_gram");
  DBuf<double>& Y3 = scratch_f64(c, "rnd_Y3");
  DBuf<double>& g = scratch_f64(c, "rnd_g");
  gram.alloc((size_t)r * r);
  Y3.alloc((size_t)n * 3);
  g.alloc(16);
  // Gram YᵀY and its top-3 eigenvectors
  k_gram<<<r * (r + 1) / 2, 256, 0, c->stream>>>(n, r, c->Y.p, gram.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  std::vector<double> hg(r * r), V, ev;
  XM_CUDA(cudaMemcpyAsync(hg.data(), gram.p, r * r * 8, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  jacobi_host(r, hg, V, ev);
  std::vector<double> W3(r * 3);
  for (int p = 0; p < r; ++p)
    for (int q = 0; q < 3; ++q) W3[p * 3 + q] = V[p * r + q];
  DBuf<double>& dW3 = scratch_f64(c, "rnd_W3");
  dW3.alloc(r * 3);
  XM_CUDA(cudaMemcpyAsync(dW3.p, W3.data(), r * 3 * 8, cudaMemcpyHostToDevice, c->stream));
  k_y_times_w3<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, r, c->Y.p, dW3.p, Y3.p);
  c->flags.alloc(16);
  XM_CUDA(cudaMemsetAsync(c->flags.p, 0, 16 * sizeof(int), c->stream));
  k_gauge0<<<1, 1, 0, c->stream>>>(Y3.p, g.p, c->flags.p + 1);
  k_round_blocks<<<ceil_div(N, 128), 128, 0, c->stream>>>(N, Y3.p, g.p, c->Rs.p, c->s_out.p, c->Yr.p,
                                                         c->flags.p, c->flags.p + 1);
  XM_CHECK_LAUNCH();
  count_launch(c, 3);
  // translations: T = −L⁻ᵀ (G Y_r), t_0 = 0
  if (c->implicit_active) {
    implicit_translations(c, c->Yr.p, c->t_out.p);  // t = −K̄⁻¹ C̄ Y₃, t_0 = 0
  } else if (N > 1 && c->have_recovery) {
    int m = N - 1;
    k_g_times_y3<<<ceil_div(m, 8), 256, 0, c->stream>>>(m, n, c->ldq, c->G.p, c->Yr.p, c->rhs.p);
    XM_CUDA(cudaMemsetAsync(c->t_out.p, 0, 3 * sizeof(double), c->stream));  // t_0 = 0
    for (int kb = ((m - 1) / kBS) * kBS; kb >= 0; kb -= kBS) {
      const int nb = std::min(kBS, m - kb);
      k_backsub_block<<<std::max(1, ceil_div(kb, 256)), 256, 0, c->stream>>>(kb, nb, c->ldk, c->L.p,
                                                                           c->rhs.p, c->t_out.p);
    }
    XM_CHECK_LAUNCH();
    count_launch(c, 1 + (m - 1) / kBS + 1);
  } else {
    XM_CUDA(cudaMemsetAsync(c->t_out.p, 0, (size_t)N * 3 * 8, c->stream));
  }
  if (c->have_recovery) {
    k_points<<<ceil_div(M, 128), 128, 0, c->stream>>>(M, c->lm_off.p, c->e_fr.p, c->e_pts.p,
                                                     c->e_w.p, c->W.p, c->Rs.p, c->s_out.p,
                                                     c->t_out.p, c->p_out.p);
    XM_CHECK_LAUNCH();
    count_launch(c);
  }
  int hf[2] = {0, 0};
  XM_CUDA(cudaMemcpyAsync(hf, c->flags.p, 8, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (hf[1]) throw Error(XM_EDEGENERATE, "degenerate block");
  c->n_flipped = hf[0];
  c->have_round = true;
}

}  // namespace xm
