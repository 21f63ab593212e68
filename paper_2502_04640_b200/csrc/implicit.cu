// implicit.cu — SURVEY §8(f) NEXT-1: Q·V without ever forming Q ("Extending
// the XM solver to support sparse matrix-vector multiplications").
//
// The two eliminations of App. A applied to V itself — the
// envelope theorem on Eq. (3): Q·V = ½∇_V min_{t,p} Σ_e w_e‖V_iᵀũ_e + t_i − p_k‖²
// (t_0 = 0).  Per product (oracle: xm_oracle.ImplicitQ):
//
//   z_e = V_iᵀ ũ_e,   m_k = Σ_{e∈k} w_e z_e / W_k           k_imp_lm_mean  (landmark pass)
//   b_i = Σ_{e∈i} w_e (z_e − m_k)          (= (C̄V)_i)        k_imp_fr_b     (frame pass)
//   t   = −K̄⁻¹ b,  t_0 = 0                                   k_imp_gemv     (dense K̄⁻¹)
//   p_k = m_k + Σ_{e∈k} w_e t_{i_e} / W_k                    k_imp_lm_p     (landmark pass)
//   (QV)_i = Σ_{e∈i} w_e ũ_e (z_e + t_i − p_k)ᵀ               k_imp_fr_out   (frame pass)
//
// Landmark passes walk the canonical (landmark-sorted) measurement arrays,
// frame passes a frame-sorted copy (both coalesced); one warp per landmark /
// frame, fixed-order warp reductions (deterministic).  Bytes per product ≈ 4
// passes over 40 B / measurement + 8(N−1)² for K̄⁻¹ (E: ≈ 1.6 GB vs 3.7 GB for
// the lower triangle of Q), and the assembly never forms S, C̄, G or Q — only
// K̄ (N × N), its Cholesky factor and inverse.
#include "frame_ops.cuh"

#include <cstdlib>

namespace xm {

namespace {
constexpr int kIT = 256;  // threads per block (8 warps)

template <int K>
__device__ __forceinline__ void warp_sum(double (&a)[K]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int q = 0; q < K; ++q) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
}

// m_k = Σ_{e∈k} w_e z_e / W_k, z_e = V_iᵀ ũ_e
template <int R>
__global__ void __launch_bounds__(kIT) k_imp_lm_mean(int M, const int32_t* __restrict__ lm_off,
                                                     const int32_t* __restrict__ e_fr,
                                                     const double* __restrict__ e_pts,
                                                     const double* __restrict__ e_w,
                                                     const double* __restrict__ W,
                                                     const double* __restrict__ V,
                                                     double* __restrict__ m,
    const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  const int k = blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= M) return;
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  for (int e = lm_off[k] + lane; e < lm_off[k + 1]; e += 32) {
    const int i = e_fr[e];
    const double u0 = e_pts[3 * e], u1 = e_pts[3 * e + 1], u2 = e_pts[3 * e + 2], we = e_w[e];
    const double* vi = V + (int64_t)3 * i * R;
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] = fma(we, fma(vi[c], u0, fma(vi[R + c], u1, vi[2 * R + c] * u2)), acc[c]);
  }
  warp_sum<R>(acc);
  if (lane == 0) {
    const double wk = W[k], inv = wk > 0.0 ? 1.0 / wk : 0.0;
#pragma unroll
    for (int c = 0; c < R; ++c) m[(int64_t)k * R + c] = acc[c] * inv;
  }
}

// b_i = Σ_{e∈i} w_e (z_e − m_k), i ≥ 1 (frame-sorted copies f_lm, f_pts, f_w)
template <int R>
__global__ void __launch_bounds__(kIT) k_imp_fr_b(int N, const int32_t* __restrict__ fr_off,
                                                  const int32_t* __restrict__ f_lm,
                                                  const double* __restrict__ f_pts,
                                                  const double* __restrict__ f_w,
                                                  const double* __restrict__ V,
                                                  const double* __restrict__ m,
                                                  double* __restrict__ b,
    const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  const int i = blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= N) return;
  double vi[3][R], acc[R];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) vi[a][c] = V[((int64_t)3 * i + a) * R + c];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  for (int q = fr_off[i] + lane; q < fr_off[i + 1]; q += 32) {
    const int k = f_lm[q];
    const double u0 = f_pts[3 * q], u1 = f_pts[3 * q + 1], u2 = f_pts[3 * q + 2], we = f_w[q];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const double z = fma(vi[0][c], u0, fma(vi[1][c], u1, vi[2][c] * u2));
      acc[c] = fma(we, z - m[(int64_t)k * R + c], acc[c]);
    }
  }
  warp_sum<R>(acc);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < R; ++c) b[(int64_t)i * R + c] = acc[c];
}

// t_{j+1} = −Σ_l Kinv[j][l] b_{l+1}  (rows j = 0..N−2), t_0 = 0
template <int R>
__global__ void __launch_bounds__(kIT) k_imp_gemv(int m_, const double* __restrict__ Kinv, int64_t ldk,
                                                  const double* __restrict__ b,
                                                  double* __restrict__ t,
    const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  const int j = blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= m_) {
    if (j == m_ && lane < R) t[lane] = 0.0;
    return;
  }
  const double* row = Kinv + (int64_t)j * ldk;  // 256-B aligned rows (ldk % 32 == 0)
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  // 16-B loads, 4 in flight per lane (2 KB per warp and round)
  const int m2 = m_ & ~1;
  int l = 2 * lane;
  for (; l + 192 < m2; l += 256) {
    double2 kv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) kv[u] = *reinterpret_cast<const double2*>(row + l + 64 * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int l0 = l + 64 * u;
#pragma unroll
      for (int c = 0; c < R; ++c)
        acc[c] = fma(kv[u].x, b[(int64_t)(l0 + 1) * R + c], fma(kv[u].y, b[(int64_t)(l0 + 2) * R + c], acc[c]));
    }
  }
  for (; l < m2; l += 64) {
    const double2 kv = *reinterpret_cast<const double2*>(row + l);
#pragma unroll
    for (int c = 0; c < R; ++c)
      acc[c] = fma(kv.x, b[(int64_t)(l + 1) * R + c], fma(kv.y, b[(int64_t)(l + 2) * R + c], acc[c]));
  }
  if (lane == 0 && (m_ & 1)) {
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] = fma(row[m_ - 1], b[(int64_t)m_ * R + c], acc[c]);
  }
  warp_sum<R>(acc);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < R; ++c) t[(int64_t)(j + 1) * R + c] = -acc[c];
}

// Symmetric K̄⁻¹ product over its LOWER triangle only (half the bytes of the
// row GEMV): CTA = one 64 × 64 tile (I, J ≤ I) of the lower triangle, 256
// threads (thread = column quarter-row...): row part  Σ_{l∈J} K[i][l] b_l  for
// its 64 rows → rowp[I][J], and (J < I) column part Σ_{i∈I} K[i][l] b_i for its
// 64 columns → colp[J][I]; k_imp_symv_fin sums a row's partials in a fixed
// order (deterministic), t = −(·).
constexpr int kST = 64;
__device__ __forceinline__ void tile_of(int64_t tt, int& I, int& J) {
  int a = (int)((sqrt(8.0 * (double)tt + 1.0) - 1.0) * 0.5);
  while ((int64_t)(a + 1) * (a + 2) / 2 <= tt) ++a;
  while ((int64_t)a * (a + 1) / 2 > tt) --a;
  I = a;
  J = (int)(tt - (int64_t)a * (a + 1) / 2);
}

// persistent: CTA c handles tiles c, c + G, …; the next tile's 8 16-B loads per
// thread are issued before the current tile is reduced (register double buffer)
template <int R>
__global__ void __launch_bounds__(256) k_imp_symv_tiles(int m_, int nb, const double* __restrict__ Kinv,
                                                         int64_t ldk, const double* __restrict__ b,
                                                         double* __restrict__ rowp,
                                                         double* __restrict__ colp,
                                                         const int* __restrict__ stop) {
  if (stop && *stop) return;
  const int64_t ntile = (int64_t)nb * (nb + 1) / 2;
  __shared__ double bJ[kST][R], bI[kST][R];
  __shared__ double red[8][kST][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = 2 * lane;
  auto load = [&](int64_t tt, double2 (&v)[8]) {
    int I, J;
    tile_of(tt, I, J);
    const int r0 = I * kST, c0 = J * kST;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int gr = r0 + warp + 8 * u, gc = c0 + q;
      v[u] = make_double2(0.0, 0.0);
      if (gr < m_ && gc + 1 < m_) v[u] = __ldcs(reinterpret_cast<const double2*>(Kinv + (int64_t)gr * ldk + gc));
      else if (gr < m_ && gc < m_) v[u].x = Kinv[(int64_t)gr * ldk + gc];
    }
  };
  double2 v[8], vn[8];
  int64_t tt = blockIdx.x;
  if (tt < ntile) load(tt, v);
  for (; tt < ntile; tt += gridDim.x) {
    const int64_t tn = tt + gridDim.x;
    if (tn < ntile) load(tn, vn);
    int I, J;
    tile_of(tt, I, J);
    const bool diag = (I == J);
    const int r0 = I * kST, c0 = J * kST;
    for (int e = threadIdx.x; e < kST * R; e += 256) {
      const int a = e / R, cc = e % R;
      bJ[a][cc] = (c0 + a < m_) ? b[(int64_t)(c0 + a + 1) * R + cc] : 0.0;
      bI[a][cc] = (r0 + a < m_) ? b[(int64_t)(r0 + a + 1) * R + cc] : 0.0;
    }
    __syncthreads();
    double cpa[R], cpb[R];
#pragma unroll
    for (int cc = 0; cc < R; ++cc) cpa[cc] = cpb[cc] = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int aa = warp + 8 * u;
      const double ka = (!diag || q <= aa) ? v[u].x : 0.0;
      const double kb = (!diag || q + 1 <= aa) ? v[u].y : 0.0;
      double rp[R];
#pragma unroll
      for (int cc = 0; cc < R; ++cc) rp[cc] = fma(ka, bJ[q][cc], kb * bJ[q + 1][cc]);
      warp_sum<R>(rp);
      if (lane == 0)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) rowp[(tt * kST + aa) * R + cc] = rp[cc];
      const double sa = (!diag || q < aa) ? v[u].x : 0.0;
      const double sb = (!diag || q + 1 < aa) ? v[u].y : 0.0;
#pragma unroll
      for (int cc = 0; cc < R; ++cc) {
        cpa[cc] = fma(sa, bI[aa][cc], cpa[cc]);
        cpb[cc] = fma(sb, bI[aa][cc], cpb[cc]);
      }
    }
#pragma unroll
    for (int c0r = 0; c0r < R; c0r += 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (c0r + k < R) {
          red[warp][q][k] = cpa[c0r + k];
          red[warp][q + 1][k] = cpb[c0r + k];
        }
      __syncthreads();
      for (int e = threadIdx.x; e < kST * 4; e += 256) {
        const int l = e >> 2, k = e & 3;
        if (c0r + k < R) {
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < 8; ++w) sum += red[w][l][k];
          colp[(tt * kST + l) * R + c0r + k] = sum;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = vn[u];
  }
}

// t_{g+1} = −( Σ_{J ≤ I} rowp[tile(I,J)][a] + Σ_{I' ≥ I} colp[tile(I',I)][a] ),  g = I·64 + a
template <int R>
__global__ void k_imp_symv_fin(int m_, int nb, const double* __restrict__ rowp,
                               const double* __restrict__ colp, double* __restrict__ t,
                               const int* __restrict__ stop) {
  if (stop && *stop) return;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e == 0)
#pragma unroll
    for (int cc = 0; cc < R; ++cc) t[cc] = 0.0;
  if (e >= (int64_t)m_ * R) return;
  const int g = (int)(e / R), cc = (int)(e % R);
  const int I = g / kST, a = g % kST;
  double s = 0.0;
  for (int J = 0; J <= I; ++J) s += rowp[(((int64_t)I * (I + 1) / 2 + J) * kST + a) * R + cc];
  for (int I2 = I; I2 < nb; ++I2) s += colp[(((int64_t)I2 * (I2 + 1) / 2 + I) * kST + a) * R + cc];
  t[(int64_t)(g + 1) * R + cc] = -s;
}

// p_k = m_k + Σ_{e∈k} w_e t_{i_e} / W_k
template <int R>
__global__ void __launch_bounds__(kIT) k_imp_lm_p(int M, const int32_t* __restrict__ lm_off,
                                                  const int32_t* __restrict__ e_fr,
                                                  const double* __restrict__ e_w,
                                                  const double* __restrict__ W,
                                                  const double* __restrict__ t,
                                                  const double* __restrict__ m,
                                                  double* __restrict__ p,
    const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  const int k = blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= M) return;
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  for (int e = lm_off[k] + lane; e < lm_off[k + 1]; e += 32) {
    const double we = e_w[e];
    const double* ti = t + (int64_t)e_fr[e] * R;
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] = fma(we, ti[c], acc[c]);
  }
  warp_sum<R>(acc);
  if (lane == 0) {
    const double wk = W[k], inv = wk > 0.0 ? 1.0 / wk : 0.0;
#pragma unroll
    for (int c = 0; c < R; ++c) p[(int64_t)k * R + c] = fma(acc[c], inv, m[(int64_t)k * R + c]);
  }
}

// (QV)_i = Σ_{e∈i} w_e ũ_e (z_e + t_i − p_k)ᵀ
template <int R>
__global__ void __launch_bounds__(kIT) k_imp_fr_out(int N, const int32_t* __restrict__ fr_off,
                                                    const int32_t* __restrict__ f_lm,
                                                    const double* __restrict__ f_pts,
                                                    const double* __restrict__ f_w,
                                                    const double* __restrict__ V,
                                                    const double* __restrict__ t,
                                                    const double* __restrict__ p,
                                                    double* __restrict__ out,
    const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  const int i = blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= N) return;
  double vi[3][R], ti[R], acc[3 * R];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) vi[a][c] = V[((int64_t)3 * i + a) * R + c];
#pragma unroll
  for (int c = 0; c < R; ++c) ti[c] = t[(int64_t)i * R + c];
#pragma unroll
  for (int q = 0; q < 3 * R; ++q) acc[q] = 0.0;
  for (int q = fr_off[i] + lane; q < fr_off[i + 1]; q += 32) {
    const int k = f_lm[q];
    const double u[3] = {f_pts[3 * q], f_pts[3 * q + 1], f_pts[3 * q + 2]};
    const double we = f_w[q];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const double z = fma(vi[0][c], u[0], fma(vi[1][c], u[1], vi[2][c] * u[2]));
      const double rr = we * (z + ti[c] - p[(int64_t)k * R + c]);
#pragma unroll
      for (int a = 0; a < 3; ++a) acc[a * R + c] = fma(u[a], rr, acc[a * R + c]);
    }
  }
  warp_sum<3 * R>(acc);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 3 * R; ++q) out[(int64_t)3 * i * R + q] = acc[q];
}

__global__ void k_frame_sorted_copy(int64_t E, const int32_t* __restrict__ fr_edge,
                                    const int32_t* __restrict__ e_lm, const double* __restrict__ e_pts,
                                    const double* __restrict__ e_w, int32_t* __restrict__ f_lm,
                                    double* __restrict__ f_pts, double* __restrict__ f_w) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= E) return;
  const int e = fr_edge[q];
  f_lm[q] = e_lm[e];
  f_pts[3 * q] = e_pts[3 * e];
  f_pts[3 * q + 1] = e_pts[3 * e + 1];
  f_pts[3 * q + 2] = e_pts[3 * e + 2];
  f_w[q] = e_w[e];
}

__global__ void k_rademacher_pack(int64_t n, int r, int col, const double* __restrict__ u,
                                  double* __restrict__ Z) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < n) Z[x * r + col] = (u[x] < 0.0) ? -1.0 : 1.0;
}

#define XM_IMP_DISPATCH(r, CALL)                                                 \
  switch (r) {                                                                   \
    case 1: { constexpr int R = 1; CALL; } break;                                \
    case 2: { constexpr int R = 2; CALL; } break;                                \
    case 3: { constexpr int R = 3; CALL; } break;                                \
    case 4: { constexpr int R = 4; CALL; } break;                                \
    case 5: { constexpr int R = 5; CALL; } break;                                \
    case 6: { constexpr int R = 6; CALL; } break;                                \
    case 7: { constexpr int R = 7; CALL; } break;                                \
    case 8: { constexpr int R = 8; CALL; } break;                                \
    case 9: { constexpr int R = 9; CALL; } break;                                \
    case 10: { constexpr int R = 10; CALL; } break;                              \
    case 11: { constexpr int R = 11; CALL; } break;                              \
    case 12: { constexpr int R = 12; CALL; } break;                              \
    default: throw Error(XM_EINVAL, "rank r out of range (1..12)");             \
  }
}  // namespace

// Matrix-free assembly state: frame-sorted measurement copies and K̄⁻¹.
void implicit_prepare(xm_ctx* c) {
  const int64_t E = c->E;
  const int N = c->N;
  c->imp_lm.alloc(E);
  c->imp_pts.alloc(3 * E);
  c->imp_w.alloc(E);
  k_frame_sorted_copy<<<ceil_div(E, 256), 256, 0, c->stream>>>(E, c->fr_edge.p, c->e_lm.p, c->e_pts.p,
                                                              c->e_w.p, c->imp_lm.p, c->imp_pts.p,
                                                              c->imp_w.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  if (N > 1) {  // K̄⁻¹ = L⁻ᵀ L⁻¹ with X = L⁻¹ (c->L, U = Lᵀ from the Cholesky)
    const int m = N - 1;
    DBuf<double>& U = scratch_f64(c, "chol_U");
    DBuf<double>& X = scratch_f64(c, "imp_X");
    X.alloc((size_t)m * c->ldk);
    identity(c, X.p, m, c->ldk);
    dense_trsm_lower_left(c, c->L.p, m, c->ldk, U.p, c->ldk, X.p, m, c->ldk);
    c->Kinv.alloc((size_t)m * c->ldk);
    // Kinv[i][j] = Σ_k X[k][i] X[k][j]  (lower tiles, then mirrored)
    dgemm_tn(c, true, m, m, m, 1.0, X.p, c->ldk, X.p, c->ldk, 0.0, c->Kinv.p, c->ldk);
    mirror_lower(c, c->Kinv.p, m, c->ldk);
  }
}

void implicit_product(xm_ctx* c, const double* V, int r, double* out, const int* stop) {
  const int N = c->N, M = c->M;
  DBuf<double>& m = scratch_f64(c, "imp_m");
  DBuf<double>& p = scratch_f64(c, "imp_p");
  DBuf<double>& b = scratch_f64(c, "imp_b");
  DBuf<double>& t = scratch_f64(c, "imp_t");
  m.alloc((size_t)M * XM_MAX_R + 8);
  p.alloc((size_t)M * XM_MAX_R + 8);
  b.alloc((size_t)N * XM_MAX_R + 8);
  t.alloc((size_t)N * XM_MAX_R + 8);
  const int gM = ceil_div(M, kIT / 32), gN = ceil_div(N, kIT / 32), gK = ceil_div(N, kIT / 32);
  XM_IMP_DISPATCH(r, (k_imp_lm_mean<R><<<gM, kIT, 0, c->stream>>>(M, c->lm_off.p, c->e_fr.p, c->e_pts.p,
                                                                  c->e_w.p, c->W.p, V, m.p, stop)));
  XM_IMP_DISPATCH(r, (k_imp_fr_b<R><<<gN, kIT, 0, c->stream>>>(N, c->fr_off.p, c->imp_lm.p, c->imp_pts.p,
                                                               c->imp_w.p, V, m.p, b.p, stop)));
  // K̄⁻¹ b: the row GEMV over the full (mirrored) K̄⁻¹ (E: 826 MB, 217 µs) is the
  // default; the lower-triangle variant (XM_IMP_SYMV=1: 415 MB + 39 MB of
  // partials) measured 195 + 37 µs — it is bound by its per-tile reductions,
  // not by the bytes (profiles/r2_implicit_E.txt)
  if (N > 1 && std::getenv("XM_IMP_SYMV")) {
    const int mK = N - 1, nb = ceil_div(mK, kST);
    const int64_t ntile = (int64_t)nb * (nb + 1) / 2;
    DBuf<double>& rp = scratch_f64(c, "imp_rowp");
    DBuf<double>& cp = scratch_f64(c, "imp_colp");
    rp.alloc((size_t)ntile * kST * XM_MAX_R + 8);
    cp.alloc((size_t)ntile * kST * XM_MAX_R + 8);
    const unsigned gsym = (unsigned)std::min<int64_t>(ntile, 148 * 8);
    XM_IMP_DISPATCH(r, (k_imp_symv_tiles<R><<<gsym, 256, 0, c->stream>>>(
                           mK, nb, c->Kinv.p, c->ldk, b.p, rp.p, cp.p, stop)));
    XM_IMP_DISPATCH(r, (k_imp_symv_fin<R><<<ceil_div((int64_t)mK * r, 256), 256, 0, c->stream>>>(
                           mK, nb, rp.p, cp.p, t.p, stop)));
    count_launch(c);
  } else if (N > 1) {
    XM_IMP_DISPATCH(r, (k_imp_gemv<R><<<gK, kIT, 0, c->stream>>>(N - 1, c->Kinv.p, c->ldk, b.p, t.p,
                                                                 stop)));
  } else {
    XM_CUDA(cudaMemsetAsync(t.p, 0, (size_t)r * 8, c->stream));
  }
  XM_IMP_DISPATCH(r, (k_imp_lm_p<R><<<gM, kIT, 0, c->stream>>>(M, c->lm_off.p, c->e_fr.p, c->e_w.p, c->W.p,
                                                               t.p, m.p, p.p, stop)));
  XM_IMP_DISPATCH(r, (k_imp_fr_out<R><<<gN, kIT, 0, c->stream>>>(N, c->fr_off.p, c->imp_lm.p,
                                                                 c->imp_pts.p, c->imp_w.p, V, t.p, p.p,
                                                                 out, stop)));
  XM_CHECK_LAUNCH();
  count_launch(c, 5);
}

// translations of the rounded solution, t = −K̄⁻¹ C̄ Y₃ (Eq. (4)), from the same passes
void implicit_translations(xm_ctx* c, const double* Y3, double* t_out) {
  const int N = c->N, M = c->M;
  DBuf<double>& m = scratch_f64(c, "imp_m");
  DBuf<double>& b = scratch_f64(c, "imp_b");
  m.alloc((size_t)M * XM_MAX_R + 8);
  b.alloc((size_t)N * XM_MAX_R + 8);
  const int gM = ceil_div(M, kIT / 32), gN = ceil_div(N, kIT / 32);
  k_imp_lm_mean<3><<<gM, kIT, 0, c->stream>>>(M, c->lm_off.p, c->e_fr.p, c->e_pts.p, c->e_w.p, c->W.p, Y3,
                                              m.p, nullptr);
  k_imp_fr_b<3><<<gN, kIT, 0, c->stream>>>(N, c->fr_off.p, c->imp_lm.p, c->imp_pts.p, c->imp_w.p, Y3, m.p,
                                           b.p, nullptr);
  if (N > 1) k_imp_gemv<3><<<gN, kIT, 0, c->stream>>>(N - 1, c->Kinv.p, c->ldk, b.p, t_out, nullptr);
  else XM_CUDA(cudaMemsetAsync(t_out, 0, 3 * 8, c->stream));
  XM_CHECK_LAUNCH();
  count_launch(c, 3);
}

// ‖Q‖_F by the shared 16-probe Rademacher estimate (reading C24; oracle
// hutchinson_normF): probe j = sign(splitmix64 stream, seed 0x48C0 + j)
double implicit_normF(xm_ctx* c) {
  constexpr int kProbes = 16, kBatch = 4;
  const int64_t n = c->n;
  DBuf<double>& Z = scratch_f64(c, "imp_probe");
  DBuf<double>& QZ = scratch_f64(c, "imp_probe_q");
  DBuf<double>& u = scratch_f64(c, "imp_probe_u");
  DBuf<double>& part = scratch_f64(c, "imp_probe_part");
  Z.alloc((size_t)n * kBatch);
  QZ.alloc((size_t)n * kBatch);
  u.alloc((size_t)n);
  part.alloc(kDotBlocks);
  double total = 0.0;
  for (int j0 = 0; j0 < kProbes; j0 += kBatch) {
    for (int q = 0; q < kBatch; ++q) {
      splitmix_uniform(c, n, 0x48C0ull + (uint64_t)(j0 + q), u.p);
      k_rademacher_pack<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, kBatch, q, u.p, Z.p);
      XM_CHECK_LAUNCH();
      count_launch(c);
    }
    implicit_product(c, Z.p, kBatch, QZ.p, nullptr);
    dot_flat(c, QZ.p, QZ.p, n * kBatch, part.p, kDotBlocks);
    reduce_partials(c, part.p, kDotBlocks, 1, c->scal.p + 30);
    double s = 0.0;
    XM_CUDA(cudaMemcpyAsync(&s, c->scal.p + 30, 8, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    total += s;
  }
  return std::sqrt(total / kProbes);
}

}  // namespace xm
