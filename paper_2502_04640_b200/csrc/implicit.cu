// implicit.cu — SURVEY §8(f) NEXT-1: Q·V without ever forming Q ("Extending
// the XM solver to support sparse matrix-vector multiplications").
//
// The two eliminations of App. A applied to V itself — the
// envelope theorem on Eq. (3): Q·V = ½∇_V min_{t,p} Σ_e w_e‖V_iᵀũ_e + t_i − p_k‖²
// (t_0 = 0).  Per product (oracle: xm_oracle.ImplicitQ):
//
//   z_e = V_iᵀ ũ_e,   m_k = Σ_{e∈k} w_e z_e / W_k           k_imp_lm_mean  (landmark pass)
//   b_i = Σ_{e∈i} w_e (z_e − m_k)          (= (C̄V)_i)        k_imp_fr_b     (frame pass)
//   t   = −K̄⁻¹ b,  t_0 = 0                                   k_spmm_sym on the lower triangle
//                                                             of K̄⁻¹ (spmm_sym.cu; r ≤ 5) or
//                                                             k_imp_gemv (full rows, r > 5)
//   p_k = m_k + Σ_{e∈k} w_e t_{i_e} / W_k                    k_imp_lm_p     (landmark pass)
//   (QV)_i = Σ_{e∈i} w_e ũ_e (z_e + t_i − p_k)ᵀ               k_imp_fr_out   (frame pass)
//
// evaluated through per-frame moments c_i = Σ_{e∈i} w_e ũ_e, A_i = Σ_{e∈i} w_e ũ_e ũ_eᵀ
// and w·ũ premultiplied per measurement (b_i = c_iᵀV_i − Σ w_e m_k;
// (QV)_i = A_iV_i + c_i t_iᵀ − Σ (wũ)_e p_kᵀ).  Landmark passes walk the canonical
// (landmark-sorted) measurement arrays, frame passes frame-sorted copies (both
// coalesced); one warp per landmark / frame, fixed-order reductions
// (deterministic).  Bytes per product: 80 B per measurement over the four passes
// + 8·m(m+1)/2 for the lower triangle of K̄⁻¹ (E: 0.81 GB vs 3.71 GB for the
// lower triangle of Q); the assembly never forms S, C̄, G or Q — only K̄
// (N × N), its Cholesky factor and inverse.  world > 1: each rank runs its
// share of every pass and a band of K̄⁻¹, one all-reduce per pass.
#include "frame_ops.cuh"

#include <algorithm>
#include <cstdio>
#include <vector>
#include <cstdlib>

namespace xm {

namespace {
constexpr int kIT = 256;  // threads per block (8 warps)
constexpr int kU = 4;     // measurements per lane in flight (ILP of the gather passes)

template <int K>
__device__ __forceinline__ void warp_sum(double (&a)[K]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int q = 0; q < K; ++q) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
}

// Every pass is one warp per landmark or frame walking its contiguous run of
// measurements in the COLUMN-OWNER layout: a group of R lanes per measurement,
// lane j of a group owning column j (⌊32/R⌋ measurements per warp round), so
// the gathered row of a measurement (V_i: 3R doubles, m_k / t_i / p_k: R
// doubles) is read by R adjacent lanes — one or two 32-B sectors per group —
// instead of one scattered sector per lane and element; the L1 wavefronts of
// the gathers, which bound these passes, drop by ≈ R×.  Each lane accumulates
// its own column; the groups are summed at the end by a fixed shuffle tree
// (deterministic).  kU rounds in flight per lane; run tails use CLAMPED
// unconditional loads with zeroed weights, never predicated loads (the
// predicated-load form of the unrolled loop faulted on sm_100a with
// data-dependent gathered addresses — DESIGN.md §5).  Per-measurement
// streams are read evict-first (__ldcs) so the gathered n × r arrays
// (≤ 1.5 MB) stay in L2.
template <int R>
struct Grp {
  static constexpr int NG = 32 / R;  // measurements per warp round
};
// row stride of the landmark arrays m and p (M × PR): r rounded up to even, so
// the frame-output pass gathers a landmark's row of p with 16-B / 32-B loads and
// a gathered row never straddles a 32-B sector for r ≤ 4 (the L1 data pipe of
// these gathers costs about one wavefront per sector touched)
template <int R>
struct PStride {
  static constexpr int PR = (R + 1) & ~1;
};

// sum over the groups of the lanes owning the same column (result in group 0)
template <int R, int K>
__device__ __forceinline__ void group_sum(double (&v)[K], int g) {
  constexpr int NG = Grp<R>::NG;
#pragma unroll
  for (int s = 1; s < NG; s <<= 1) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const double o = __shfl_down_sync(0xffffffffu, v[q], s * R);
      if ((g % (2 * s)) == 0 && g + s < NG) v[q] += o;
    }
  }
}

// Frame-block transpose of V for the landmark-mean gather (r ≤ 8): frame i's
// block holds column j of V_i (3 rows + one pad) in the 32 B at Vt[i·FS + 4j],
// blocks FS doubles apart (128 B for r ≤ 4, 256 B for r ≤ 8, line-aligned), so
// the lane owning column j fetches its three values with ONE 256-bit load and a
// measurement's R lanes touch one 128-B line (three sectors, one instruction)
// instead of three row gathers straddling sectors; the L1 data pipe that bounds
// this pass costs about one wavefront per sector touched (E, r = 3: 79 → 69 µs
// with the 2-µs transpose).  Same products, same order: bitwise identical.
template <int R>
struct VtStride {
  static constexpr int FS = ((4 * R + 15) / 16) * 16;
};
constexpr int kVtMaxR = 8;

template <int R>
__global__ void k_imp_vt(int N, const double* __restrict__ V, double* __restrict__ Vt,
                         const int* __restrict__ stop) {
  if (stop && *stop) return;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;  // (frame i, column j)
  if (x >= N * R) return;
  const int i = x / R, j = x - i * R;
  const double* vi = V + (int64_t)3 * i * R + j;
  double* o = Vt + (int64_t)i * VtStride<R>::FS + 4 * j;
  o[0] = vi[0];
  o[1] = vi[R];
  o[2] = vi[2 * R];
  o[3] = 0.0;
}

__device__ __forceinline__ double4 ldg_v4(const double* p) {  // LDG.E.ENL2.256, 32-B aligned
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// m_k = Σ_{e∈k} (w_e ũ_e)ᵀ V_{i_e} / W_k          (landmark-sorted, 28 B / measurement)
// VT: V given as the frame-block transpose Vt (k_imp_vt)
template <int R, int U = kU, bool VT = false>
__global__ void __launch_bounds__(kIT) k_imp_lm_mean(int k0, int k1, const int32_t* __restrict__ lm_off,
                                                     const int32_t* __restrict__ L_i,
                                                     const double* __restrict__ L_wx,
                                                     const double* __restrict__ L_wy,
                                                     const double* __restrict__ L_wz,
                                                     const double* __restrict__ W,
                                                     const double* __restrict__ V,
                                                     double* __restrict__ m,
                                                     const int* __restrict__ stop,
                                                     int* __restrict__ exec) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  if (exec && blockIdx.x == 0 && threadIdx.x == 0) *exec = 1;  // profiling: this product ran
  constexpr int NG = Grp<R>::NG;
  const int k = k0 + blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= k1) return;
  const int g = lane / R, j = lane - g * R;
  const bool act = g < NG;
  double acc[1] = {0.0};
  const int lo = lm_off[k], hi = lm_off[k + 1];
  for (int base = lo; base < hi; base += NG * U) {
    int ii[U];
    double a0[U], a1[U], a2[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e0 = base + q * NG + g;
      const int e = min(e0, hi - 1);  // clamped: loads unconditional, tail weights zeroed
      const double okw = (act && e0 < hi) ? 1.0 : 0.0;
      ii[q] = __ldcs(L_i + e);
      a0[q] = okw * __ldcs(L_wx + e);
      a1[q] = okw * __ldcs(L_wy + e);
      a2[q] = okw * __ldcs(L_wz + e);
    }
    if constexpr (VT) {
      double4 vv[U];
#pragma unroll
      for (int q = 0; q < U; ++q) vv[q] = ldg_v4(V + (int64_t)ii[q] * VtStride<R>::FS + 4 * j);
#pragma unroll
      for (int q = 0; q < U; ++q) acc[0] = fma(a0[q], vv[q].x, fma(a1[q], vv[q].y, fma(a2[q], vv[q].z, acc[0])));
    } else {
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const double* vi = V + (int64_t)3 * ii[q] * R + j;
        acc[0] = fma(a0[q], vi[0], fma(a1[q], vi[R], fma(a2[q], vi[2 * R], acc[0])));
      }
    }
  }
  group_sum<R, 1>(acc, g);
  if (lane < R) {
    const double sum = acc[0];
    const double wk = W[k], inv = wk > 0.0 ? 1.0 / wk : 0.0;
    m[(int64_t)k * PStride<R>::PR + lane] = sum * inv;
  }
}

// b_i = Σ_{e∈i} w_e (z_e − m_k) = c_iᵀ V_i − Σ_{e∈i} w_e m_k  (c_i = Σ_{e∈i} w_e ũ_e),
// i ≥ 1, written to bs[i − 1] (the K̄ ordering: the anchor row is dropped)
// (frame-sorted, 12 B / measurement)
template <int R, int U = kU>
__global__ void __launch_bounds__(kIT) k_imp_fr_b(int f0, int f1, const int32_t* __restrict__ fr_off,
                                                  const int32_t* __restrict__ F_k,
                                                  const double* __restrict__ F_w,
                                                  const double* __restrict__ cfr,
                                                  const double* __restrict__ V,
                                                  const double* __restrict__ m,
                                                  double* __restrict__ bs,
                                                  const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  constexpr int NG = Grp<R>::NG;
  const int i = max(f0, 1) + blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= f1) return;
  const int g = lane / R, j = lane - g * R;
  const bool act = g < NG;
  double acc[1] = {0.0};
  const int lo = fr_off[i], hi = fr_off[i + 1];
  for (int base = lo; base < hi; base += NG * U) {
    int kk[U];
    double we[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e0 = base + q * NG + g;
      const int e = min(e0, hi - 1);
      kk[q] = __ldcs(F_k + e);
      we[q] = ((act && e0 < hi) ? 1.0 : 0.0) * __ldcs(F_w + e);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) acc[0] = fma(we[q], m[(int64_t)kk[q] * PStride<R>::PR + j], acc[0]);
  }
  group_sum<R, 1>(acc, g);
  if (lane < R) {
    const double sum = acc[0];
    const int jj = lane;
    const double* vi = V + (int64_t)3 * i * R + jj;
    const double* ci = cfr + 3 * (int64_t)i;
    bs[(int64_t)(i - 1) * R + jj] = fma(ci[0], vi[0], fma(ci[1], vi[R], ci[2] * vi[2 * R])) - sum;
  }
}

// Row GEMV over the full (mirrored) K̄⁻¹ for r > 5 (the lower-triangle stream
// of spmm_sym.cu covers r ≤ 5):  tb[j + 1] = Σ_l K̄⁻¹[j][l] bs[l]  (tb[0] = 0;
// the translations are t_i = −tb[i])
template <int R>
__global__ void __launch_bounds__(kIT) k_imp_gemv(int m_, int j0, int j1, const double* __restrict__ Kinv,
                                                  int64_t ldk, const double* __restrict__ bs,
                                                  double* __restrict__ tb,
                                                  const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  const int j = j0 + blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= j1) return;
  const double* row = Kinv + (int64_t)j * ldk;  // 256-B aligned rows (ldk % 32 == 0)
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  const int m2 = m_ & ~1;
  int l = 2 * lane;
  for (; l + 192 < m2; l += 256) {
    double2 kv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) kv[u] = __ldcs(reinterpret_cast<const double2*>(row + l + 64 * u));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int l0 = l + 64 * u;
#pragma unroll
      for (int c = 0; c < R; ++c)
        acc[c] = fma(kv[u].x, bs[(int64_t)l0 * R + c], fma(kv[u].y, bs[(int64_t)(l0 + 1) * R + c], acc[c]));
    }
  }
  for (; l < m2; l += 64) {
    const double2 kv = *reinterpret_cast<const double2*>(row + l);
#pragma unroll
    for (int c = 0; c < R; ++c)
      acc[c] = fma(kv.x, bs[(int64_t)l * R + c], fma(kv.y, bs[(int64_t)(l + 1) * R + c], acc[c]));
  }
  if (lane == 0 && (m_ & 1)) {
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] = fma(row[m_ - 1], bs[(int64_t)(m_ - 1) * R + c], acc[c]);
  }
  warp_sum<R>(acc);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < R; ++c) tb[(int64_t)(j + 1) * R + c] = acc[c];
}

// p_k = m_k + Σ_{e∈k} w_e t_{i_e} / W_k = m_k − Σ_{e∈k} w_e tb_{i_e} / W_k
// (landmark-sorted, 12 B / measurement)
template <int R, int U = kU>
__global__ void __launch_bounds__(kIT) k_imp_lm_p(int k0, int k1, const int32_t* __restrict__ lm_off,
                                                  const int32_t* __restrict__ L_i,
                                                  const double* __restrict__ L_w,
                                                  const double* __restrict__ W,
                                                  const double* __restrict__ tb,
                                                  const double* __restrict__ m,
                                                  double* __restrict__ p,
                                                  const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  constexpr int NG = Grp<R>::NG;
  const int k = k0 + blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= k1) return;
  const int g = lane / R, j = lane - g * R;
  const bool act = g < NG;
  double acc[1] = {0.0};
  const int lo = lm_off[k], hi = lm_off[k + 1];
  for (int base = lo; base < hi; base += NG * U) {
    int ii[U];
    double we[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e0 = base + q * NG + g;
      const int e = min(e0, hi - 1);
      ii[q] = __ldcs(L_i + e);
      we[q] = ((act && e0 < hi) ? 1.0 : 0.0) * __ldcs(L_w + e);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const double wq = (ii[q] != 0) ? we[q] : 0.0;  // t_0 = 0 (anchor)
      acc[0] = fma(wq, tb[(int64_t)ii[q] * R + j], acc[0]);
    }
  }
  group_sum<R, 1>(acc, g);
  if (lane < R) {
    const double sum = acc[0];
    const double wk = W[k], inv = wk > 0.0 ? 1.0 / wk : 0.0;
    p[(int64_t)k * PStride<R>::PR + lane] = fma(-sum, inv, m[(int64_t)k * PStride<R>::PR + lane]);
    if (PStride<R>::PR != R && lane == R - 1) p[(int64_t)k * PStride<R>::PR + R] = 0.0;
  }
}

// (QV)_i = Σ_{e∈i} w_e ũ_e (z_e + t_i − p_k)ᵀ = A_i V_i + c_i t_iᵀ − Σ_{e∈i} (w_e ũ_e) p_kᵀ
// (A_i = Σ_{e∈i} w_e ũ_e ũ_eᵀ, t_i = −tb_i; frame-sorted, 28 B / measurement)
template <int R, int U = ((R <= 3) ? 4 : 2)>
__global__ void __launch_bounds__(kIT, (R <= 5) ? 4 : 1) k_imp_fr_out(int f0, int f1, const int32_t* __restrict__ fr_off,
                                                    const int32_t* __restrict__ F_k,
                                                    const double* __restrict__ F_wx,
                                                    const double* __restrict__ F_wy,
                                                    const double* __restrict__ F_wz,
                                                    const double* __restrict__ cfr,
                                                    const double* __restrict__ Afr,
                                                    const double* __restrict__ V,
                                                    const double* __restrict__ tb,
                                                    const double* __restrict__ p,
                                                    double* __restrict__ out,
                                                    const int* __restrict__ stop) {
  if (stop && *stop) return;  // a tCG graph replay past the stop
  const int i = f0 + blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= f1) return;
  double acc[3 * R];
#pragma unroll
  for (int q = 0; q < 3 * R; ++q) acc[q] = 0.0;
  const int lo = fr_off[i], hi = fr_off[i + 1];
  for (int q0 = lo + lane; q0 < hi; q0 += 32 * U) {
    int kk[U];
    double a0[U], a1[U], a2[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e = min(q0 + 32 * q, hi - 1);
      const double okw = (q0 + 32 * q < hi) ? 1.0 : 0.0;
      kk[q] = __ldcs(F_k + e);
      a0[q] = okw * __ldcs(F_wx + e);
      a1[q] = okw * __ldcs(F_wy + e);
      a2[q] = okw * __ldcs(F_wz + e);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      constexpr int PR = PStride<R>::PR;
      double pv[PR];
      if constexpr (PR % 4 == 0) {  // 256-bit loads (32-B aligned rows): one access per 4 values
#pragma unroll
        for (int h = 0; h < PR / 4; ++h) {
          const double4 t4 = ldg_v4(p + (int64_t)kk[q] * PR + 4 * h);
          pv[4 * h] = t4.x;
          pv[4 * h + 1] = t4.y;
          pv[4 * h + 2] = t4.z;
          pv[4 * h + 3] = t4.w;
        }
      } else {
        const double2* pk = reinterpret_cast<const double2*>(p + (int64_t)kk[q] * PR);
#pragma unroll
        for (int h = 0; h < PR / 2; ++h) {
          const double2 t2 = pk[h];
          pv[2 * h] = t2.x;
          pv[2 * h + 1] = t2.y;
        }
      }
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const double pc = pv[c];
        acc[c] = fma(a0[q], pc, acc[c]);
        acc[R + c] = fma(a1[q], pc, acc[R + c]);
        acc[2 * R + c] = fma(a2[q], pc, acc[2 * R + c]);
      }
    }
  }
  warp_sum<3 * R>(acc);
#pragma unroll
  for (int l0 = 0; l0 < 3 * R; l0 += 32) {  // 3R > 32 for r ≥ 11
    const int x = l0 + lane;
    if (x >= 3 * R) break;
    const int a = x / R, c = x % R;
    double s = acc[l0];
#pragma unroll
    for (int q = l0 + 1; q < 3 * R && q < l0 + 32; ++q) s = (x == q) ? acc[q] : s;
    const double* Ai = Afr + 6 * (int64_t)i;  // xx yy zz xy xz yz
    const double A0 = a == 0 ? Ai[0] : (a == 1 ? Ai[3] : Ai[4]);
    const double A1 = a == 0 ? Ai[3] : (a == 1 ? Ai[1] : Ai[5]);
    const double A2 = a == 0 ? Ai[4] : (a == 1 ? Ai[5] : Ai[2]);
    const double* vi = V + (int64_t)3 * i * R + c;
    const double av = fma(A0, vi[0], fma(A1, vi[R], A2 * vi[2 * R]));
    const double tbi = (i > 0) ? tb[(int64_t)i * R + c] : 0.0;  // t_0 = 0 (anchor)
    out[(int64_t)3 * i * R + x] = fma(-cfr[3 * (int64_t)i + a], tbi, av) - s;
  }
}

// Matrix-free layout (once per build): landmark-sorted w·ũ (SoA), the
// frame-sorted landmark ids, weights and w·ũ (SoA).
__global__ void k_imp_layout(int64_t E, const int32_t* __restrict__ fr_edge,
                             const int32_t* __restrict__ e_lm, const double* __restrict__ e_pts,
                             const double* __restrict__ e_w, double* __restrict__ L_wx,
                             double* __restrict__ L_wy, double* __restrict__ L_wz,
                             int32_t* __restrict__ F_k, double* __restrict__ F_w,
                             double* __restrict__ F_wx, double* __restrict__ F_wy,
                             double* __restrict__ F_wz) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= E) return;
  {
    const double w = e_w[q];
    L_wx[q] = w * e_pts[3 * q];
    L_wy[q] = w * e_pts[3 * q + 1];
    L_wz[q] = w * e_pts[3 * q + 2];
  }
  const int e = fr_edge[q];
  const double w = e_w[e];
  F_k[q] = e_lm[e];
  F_w[q] = w;
  F_wx[q] = w * e_pts[3 * e];
  F_wy[q] = w * e_pts[3 * e + 1];
  F_wz[q] = w * e_pts[3 * e + 2];
}

// Per-frame moments c_i = Σ_{e∈i} w_e ũ_e and A_i = Σ_{e∈i} w_e ũ_e ũ_eᵀ
// (xx yy zz xy xz yz); warp per frame, fixed order
__global__ void __launch_bounds__(kIT) k_imp_frame_moments(int N, const int32_t* __restrict__ fr_off,
                                                           const int32_t* __restrict__ fr_edge,
                                                           const double* __restrict__ e_pts,
                                                           const double* __restrict__ e_w,
                                                           double* __restrict__ cfr,
                                                           double* __restrict__ Afr) {
  const int i = blockIdx.x * (kIT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= N) return;
  double a[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) a[q] = 0.0;
  for (int q = fr_off[i] + lane; q < fr_off[i + 1]; q += 32) {
    const int e = fr_edge[q];
    const double w = e_w[e], u0 = e_pts[3 * e], u1 = e_pts[3 * e + 1], u2 = e_pts[3 * e + 2];
    a[0] = fma(w, u0, a[0]);
    a[1] = fma(w, u1, a[1]);
    a[2] = fma(w, u2, a[2]);
    a[3] = fma(w * u0, u0, a[3]);
    a[4] = fma(w * u1, u1, a[4]);
    a[5] = fma(w * u2, u2, a[5]);
    a[6] = fma(w * u0, u1, a[6]);
    a[7] = fma(w * u0, u2, a[7]);
    a[8] = fma(w * u1, u2, a[8]);
  }
  warp_sum<9>(a);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 3; ++q) cfr[3 * (int64_t)i + q] = a[q];
#pragma unroll
    for (int q = 0; q < 6; ++q) Afr[6 * (int64_t)i + q] = a[3 + q];
  }
}

// t_i = −tb_i (the rounded solution's translations, t_0 = 0)
__global__ void k_imp_neg(int64_t n, const double* __restrict__ tb, double* __restrict__ t) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < n) t[x] = (x < 3) ? 0.0 : -tb[x];
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

// the transpose and the landmark-mean pass over it (r ≤ kVtMaxR)
template <int R>
static void lm_mean_vt(xm_ctx* c, int k0, int k1, const double* V, double* vt, double* m, const int* stop,
                       int* exec) {
  if constexpr (R <= kVtMaxR) {
    const int64_t E = c->E;
    const double* P = c->imp_pts.p;
    k_imp_vt<R><<<ceil_div(c->N * R, 256), 256, 0, c->stream>>>(c->N, V, vt, stop);
    k_imp_lm_mean<R, kU, true><<<ceil_div(k1 - k0, kIT / 32), kIT, 0, c->stream>>>(
        k0, k1, c->lm_off.p, c->e_fr.p, P, P + E, P + 2 * E, c->W.p, vt, m, stop, exec);
  }
}

// XM_IMP_DEBUG=1: synchronise after every pass and name the failing one
static void imp_dbg(xm_ctx* c, const char* what) {
  static const bool on = std::getenv("XM_IMP_DEBUG") != nullptr;
  if (!on) return;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(XM_ECUDA, std::string("implicit pass ") + what + ": " + cudaGetErrorString(e));
}

static void implicit_shards(xm_ctx* c);

// Matrix-free assembly state: the pass layouts, per-frame moments and K̄⁻¹.
void implicit_prepare(xm_ctx* c) {
  const int64_t E = c->E;
  const int N = c->N;
  implicit_shards(c);
  c->imp_lm.alloc(E);
  c->imp_w.alloc(E);
  c->imp_pts.alloc(6 * E);           // L_wx L_wy L_wz F_wx F_wy F_wz
  c->imp_mom.alloc(9 * (size_t)N);   // c_i (N × 3), A_i (N × 6)
  double* P = c->imp_pts.p;
  k_imp_layout<<<ceil_div(E, 256), 256, 0, c->stream>>>(E, c->fr_edge.p, c->e_lm.p, c->e_pts.p, c->e_w.p,
                                                         P, P + E, P + 2 * E, c->imp_lm.p, c->imp_w.p,
                                                         P + 3 * E, P + 4 * E, P + 5 * E);
  imp_dbg(c, "layout");
  k_imp_frame_moments<<<ceil_div(N, kIT / 32), kIT, 0, c->stream>>>(N, c->fr_off.p, c->fr_edge.p, c->e_pts.p,
                                                                    c->e_w.p, c->imp_mom.p,
                                                                    c->imp_mom.p + 3 * (size_t)N);
  XM_CHECK_LAUNCH();
  imp_dbg(c, "moments");
  count_launch(c, 2);
  // tb = [0; K̄⁻¹ bs] with room for the padded rows of the lower-triangle stream
  c->imp_tb.alloc((size_t)(3 * ceil_div(N, 3) + 6) * XM_MAX_R + 8);
  XM_CUDA(cudaMemsetAsync(c->imp_tb.p, 0, c->imp_tb.n * 8, c->stream));
  if (N > 1) {  // K̄⁻¹ = L⁻ᵀ L⁻¹ with X = L⁻¹ (c->L, U = Lᵀ from the Cholesky)
    const int m = N - 1;
    DBuf<double>& U = scratch_f64(c, "chol_U");
    DBuf<double>& X = scratch_f64(c, "imp_X");
    X.alloc((size_t)m * c->ldk);
    identity(c, X.p, m, c->ldk);
    dense_trsm_lower_left(c, c->L.p, m, c->ldk, U.p, c->ldk, X.p, m, c->ldk, true);  // X lower triangular
    c->Kinv.alloc((size_t)m * c->ldk);
    // Kinv[i][j] = Σ_{k ≥ max(i,j)} X[k][i] X[k][j]  (lower tiles, then mirrored for the r > 5
    // row GEMV); X stays allocated (scratch): freeing and re-allocating 0.8 GB per build cost
    // up to 0.3 s of cudaFree / cudaMalloc at E
    dsyrk_tn_lowtri(c, m, 1.0, X.p, c->ldk, 0.0, c->Kinv.p, c->ldk);
    mirror_lower(c, c->Kinv.p, m, c->ldk);
    imp_dbg(c, "K^-1");
  }
}

// world > 1 (SURVEY §8(e) for the matrix-free products): every rank holds all
// measurements, the per-frame moments and the full K̄⁻¹ (as on one GPU), and
// computes its share of each pass — landmarks [k0, k1) and frames [f0, f1)
// balanced by measurement count, the K̄⁻¹ rows [ka, kb) of an area-balanced,
// 32-row-aligned band of its lower triangle — then ONE all-reduce of the
// zero-padded pass output (m, b, t, p, Q·V: ≤ 1.2 MB each at E) gives every
// rank the replicated result: five all-reduces per product, no other exchange.
static void implicit_shards(xm_ctx* c) {
  const int P = c->world, q = c->rank, N = c->N, M = c->M;
  const int64_t E = c->E;
  if (P <= 1) {
    c->imp_k0 = 0, c->imp_k1 = M, c->imp_f0 = 0, c->imp_f1 = N, c->imp_ka = 0, c->imp_kb = std::max(N - 1, 0);
    c->imp_el = c->imp_ef = E;
    return;
  }
  std::vector<int32_t> lo(M + 1), fo(N + 1);
  XM_CUDA(cudaMemcpy(lo.data(), c->lm_off.p, (M + 1) * 4, cudaMemcpyDeviceToHost));
  XM_CUDA(cudaMemcpy(fo.data(), c->fr_off.p, (N + 1) * 4, cudaMemcpyDeviceToHost));
  auto split = [&](const std::vector<int32_t>& off, int cnt, int p) {  // first segment at ≥ E·p/P
    if (p <= 0) return 0;
    if (p >= P) return cnt;
    const int64_t target = E * p / P;
    return (int)(std::lower_bound(off.begin(), off.begin() + cnt, (int32_t)target) - off.begin());
  };
  c->imp_k0 = split(lo, M, q);
  c->imp_k1 = std::max(c->imp_k0, split(lo, M, q + 1));
  c->imp_f0 = split(fo, N, q);
  c->imp_f1 = std::max(c->imp_f0, split(fo, N, q + 1));
  const int m = std::max(N - 1, 0);
  c->imp_ka = band_start(m, P, q);
  c->imp_kb = std::max(c->imp_ka, band_start(m, P, q + 1));
  c->imp_el = lo[c->imp_k1] - lo[c->imp_k0];
  c->imp_ef = fo[c->imp_f1] - fo[c->imp_f0];
}

// tb[1..N) = K̄⁻¹ bs: the lower-triangle stream (r ≤ 5; on world > 1 this rank's
// band of rows, all-reduced by the caller) or the full row GEMV.  Row 0 of tb is
// never read as data (t_0 = 0 is applied by the readers: a product at another r
// leaves other values there)
static void kinv_product(xm_ctx* c, const double* bs, int r, const int* stop, bool local_full = false) {
  const int mK = c->N - 1;
  if (mK < 1) return;  // tb stays 0 (N = 1)
  static const bool force_gemv = std::getenv("XM_IMP_GEMV") != nullptr;
  if (r <= 5 && !force_gemv && !local_full) {
    const int ka = c->world > 1 ? c->imp_ka : 0, kb = c->world > 1 ? c->imp_kb : mK;
    if (c->world > 1 && kb <= ka) {  // empty band: a zero partial
      XM_CUDA(cudaMemsetAsync(c->imp_tb.p + r, 0, (size_t)mK * r * 8, c->stream));
      return;
    }
    spmm_sym_matrix(c, c->imp_sym_plan, c->imp_sym_part, c->Kinv.p, mK, c->ldk, bs, r, c->imp_tb.p + r,
                    stop, ka, kb - ka);
  } else {  // full rows; world > 1 (r > 5): this rank's rows only, the others zero for the all-reduce
    const bool part = c->world > 1 && !local_full;
    const int j0 = part ? c->imp_ka : 0, j1 = part ? c->imp_kb : mK;
    if (part) XM_CUDA(cudaMemsetAsync(c->imp_tb.p + r, 0, (size_t)mK * r * 8, c->stream));
    if (j1 > j0)
      XM_IMP_DISPATCH(r, (k_imp_gemv<R><<<ceil_div(j1 - j0, kIT / 32), kIT, 0, c->stream>>>(
                             mK, j0, j1, c->Kinv.p, c->ldk, bs, c->imp_tb.p, stop)));
    XM_CHECK_LAUNCH();
    count_launch(c);
  }
}

// Algorithmic bytes of one matrix-free product: the four passes'
// per-measurement streams (28 + 12 + 12 + 28 B), the lower triangle of K̄⁻¹
// (r ≤ 5; the full matrix for the row GEMV) and V in / Q·V out; the gathered
// n × r / M × r arrays are L2-resident and not counted.  Per rank on world > 1.
double implicit_alg_bytes(xm_ctx* c, int r) {
  // this rank's share: its landmarks' and frames' measurements, its band of K̄⁻¹
  const double a = c->imp_ka, b = c->imp_kb;
  const double kb = (r <= 5) ? 8.0 * ((b * (b + 1.0)) - (a * (a + 1.0))) / 2.0 : 8.0 * (b - a) * ((double)c->N - 1.0);
  return 40.0 * (double)c->imp_el + 40.0 * (double)c->imp_ef + kb + 16.0 * (double)c->n * r;
}

void implicit_product(xm_ctx* c, const double* V, int r, double* out, const int* stop, int* exec) {
  const int N = c->N, M = c->M;
  const int64_t E = c->E;
  const bool sh = c->world > 1;
  DBuf<double>& m = scratch_f64(c, "imp_m");
  DBuf<double>& p = scratch_f64(c, "imp_p");
  DBuf<double>& bs = scratch_f64(c, "imp_bs");
  m.alloc((size_t)M * XM_MAX_R + 8);
  p.alloc((size_t)M * XM_MAX_R + 8);
  bs.alloc((size_t)(3 * ceil_div(N, 3) + 6) * XM_MAX_R + 8);
  const double* P = c->imp_pts.p;
  const double* cfr = c->imp_mom.p;
  const double* Afr = c->imp_mom.p + 3 * (size_t)N;
  const int k0 = c->imp_k0, k1 = c->imp_k1, f0 = c->imp_f0, f1 = c->imp_f1;
  const int PR = (r + 1) & ~1;  // m's and p's row stride (PStride)
  imp_dbg(c, "entry");
  if (sh) XM_CUDA(cudaMemsetAsync(m.p, 0, (size_t)M * PR * 8, c->stream));
  static const bool no_vt = std::getenv("XM_IMP_NO_VT") != nullptr;
  if (k1 > k0 && r <= kVtMaxR && !no_vt) {
    DBuf<double>& vt = scratch_f64(c, "imp_vt");
    vt.alloc((size_t)N * VtStride<kVtMaxR>::FS + 8);
    XM_IMP_DISPATCH(r, (lm_mean_vt<R>(c, k0, k1, V, vt.p, m.p, stop, exec)));
    count_launch(c);
  } else if (k1 > k0) {
    XM_IMP_DISPATCH(r, (k_imp_lm_mean<R><<<ceil_div(k1 - k0, kIT / 32), kIT, 0, c->stream>>>(
                           k0, k1, c->lm_off.p, c->e_fr.p, P, P + E, P + 2 * E, c->W.p, V, m.p, stop, exec)));
  }
  if (sh) nccl_allreduce_sum(c, m.p, (size_t)M * PR);
  imp_dbg(c, "lm_mean");
  const int fb0 = std::max(f0, 1);
  if (sh) XM_CUDA(cudaMemsetAsync(bs.p, 0, (size_t)std::max(N - 1, 1) * r * 8, c->stream));
  // 16 rounds in flight (E: 43 → 36 µs; the other passes measured flat or slower; two
  // frames per warp interleaved, to run the 10155 frames in one wave, measured slower: 43 vs 41 µs)
  if (f1 > fb0)
    XM_IMP_DISPATCH(r, (k_imp_fr_b<R, 16><<<ceil_div(f1 - fb0, kIT / 32), kIT, 0, c->stream>>>(
                           f0, f1, c->fr_off.p, c->imp_lm.p, c->imp_w.p, cfr, V, m.p, bs.p, stop)));
  XM_CHECK_LAUNCH();
  if (sh && N > 1) nccl_allreduce_sum(c, bs.p, (size_t)(N - 1) * r);
  imp_dbg(c, "fr_b");
  kinv_product(c, bs.p, r, stop);
  if (sh && N > 1) nccl_allreduce_sum(c, c->imp_tb.p + r, (size_t)(N - 1) * r);
  imp_dbg(c, "kinv");
  if (sh) XM_CUDA(cudaMemsetAsync(p.p, 0, (size_t)M * PR * 8, c->stream));
  if (k1 > k0)
    XM_IMP_DISPATCH(r, (k_imp_lm_p<R><<<ceil_div(k1 - k0, kIT / 32), kIT, 0, c->stream>>>(
                           k0, k1, c->lm_off.p, c->e_fr.p, c->e_w.p, c->W.p, c->imp_tb.p, m.p, p.p, stop)));
  if (sh) nccl_allreduce_sum(c, p.p, (size_t)M * PR);
  imp_dbg(c, "lm_p");
  if (sh) XM_CUDA(cudaMemsetAsync(out, 0, (size_t)3 * N * r * 8, c->stream));
  if (f1 > f0)
    XM_IMP_DISPATCH(r, (k_imp_fr_out<R><<<ceil_div(f1 - f0, kIT / 32), kIT, 0, c->stream>>>(
                           f0, f1, c->fr_off.p, c->imp_lm.p, P + 3 * E, P + 4 * E, P + 5 * E, cfr, Afr, V,
                           c->imp_tb.p, p.p, out, stop)));
  XM_CHECK_LAUNCH();
  if (sh) nccl_allreduce_sum(c, out, (size_t)3 * N * r);
  imp_dbg(c, "fr_out");
  count_launch(c, N > 1 ? 4 : 3);
}

// translations of the rounded solution, t = −K̄⁻¹ C̄ Y₃ (Eq. (4)), from the same passes
// (one-shot: every rank runs them over all landmarks / frames, no exchange)
void implicit_translations(xm_ctx* c, const double* Y3, double* t_out) {
  const int N = c->N, M = c->M;
  const int64_t E = c->E;
  DBuf<double>& m = scratch_f64(c, "imp_m");
  DBuf<double>& bs = scratch_f64(c, "imp_bs");
  m.alloc((size_t)M * XM_MAX_R + 8);
  bs.alloc((size_t)(3 * ceil_div(N, 3) + 6) * XM_MAX_R + 8);
  const double* P = c->imp_pts.p;
  k_imp_lm_mean<3><<<ceil_div(M, kIT / 32), kIT, 0, c->stream>>>(0, M, c->lm_off.p, c->e_fr.p, P, P + E,
                                                                 P + 2 * E, c->W.p, Y3, m.p, nullptr, nullptr);
  if (N > 1)
    k_imp_fr_b<3, 16><<<ceil_div(N - 1, kIT / 32), kIT, 0, c->stream>>>(0, N, c->fr_off.p, c->imp_lm.p,
                                                                        c->imp_w.p, c->imp_mom.p, Y3, m.p,
                                                                        bs.p, nullptr);
  XM_CHECK_LAUNCH();
  kinv_product(c, bs.p, 3, nullptr, c->world > 1);  // world > 1: the full-row GEMV (band plan is partial)
  k_imp_neg<<<ceil_div((int64_t)3 * N, 256), 256, 0, c->stream>>>((int64_t)3 * N, c->imp_tb.p, t_out);
  XM_CHECK_LAUNCH();
  count_launch(c, N > 1 ? 3 : 2);
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
