// assembly.cu — SURVEY §8(a) rows H1–H5 on the device.
//
//  H1 validate + de-duplicate (keep first duplicate)
//  H2 sort edges by (landmark, frame) and (frame, landmark), track stats W_k
//     (Q_3 = diag(W_k), App. A)
//  H3 co-visibility pattern of S (BSR rowptr / colidx, bit-exact contract)
//  H4 landmark elimination: row-owned clique scatter into dense S, C, K
//       H_(i,j) = Σ_k [δ_ij w_e a_e a_eᵀ − (w_e w_f / W_k) a_e a_fᵀ],  a = [ũ; 1]
//     (the expanded quadratic form of App. A P:1162-1189 with p eliminated)
//  H5 translation elimination with t_0 = 0: K̄ = L Lᵀ, G = L⁻¹ C̄,
//     Q = S − Gᵀ G  (Prop. 1 Q, P:1249 with the sign reading C1)
//
// Everything is deterministic: sorts are stable, every dense entry is owned by
// one CTA that accumulates landmarks in ascending order.
#include "xm_internal.cuh"

#include <chrono>
#include <cmath>
#include <cstdlib>

namespace xm {

// =============================================================== H1 validate
enum { ERR_RANGE = 1, ERR_WEIGHT = 2, ERR_POINT = 4 };

__global__ void k_validate(int64_t E, int N, int M, const int32_t* __restrict__ fr,
                           const int32_t* __restrict__ lm, const double* __restrict__ pts,
                           const double* __restrict__ w, int* __restrict__ err,
                           uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  int f = fr[e], k = lm[e];
  int bad = 0;
  if (f < 0 || f >= N || k < 0 || k >= M) bad |= ERR_RANGE;
  double we = w ? w[e] : 1.0;
  if (!(we > 0.0) || !isfinite(we)) bad |= ERR_WEIGHT;
  double x = pts[3 * e], y = pts[3 * e + 1], z = pts[3 * e + 2];
  if (!isfinite(x) || !isfinite(y) || !isfinite(z) || !(z > 0.0)) bad |= ERR_POINT;
  if (bad) atomicOr(err, bad);
  key[e] = bad ? 0ull : (uint64_t)f * (uint64_t)M + (uint64_t)k;  // (frame, landmark) order
  val[e] = (uint32_t)e;
}

__global__ void k_first_flags(const uint64_t* __restrict__ key, int64_t n, int32_t* __restrict__ flag) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  flag[j] = (j == 0 || key[j] != key[j - 1]) ? 1 : 0;
}

// kept frame-sorted items → (landmark, frame) keys for the second sort
__global__ void k_compact_fs(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val,
                             const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                             int64_t n, int M, int N, int32_t* __restrict__ fs_in,
                             int32_t* __restrict__ fs_fr, uint64_t* __restrict__ key2,
                             uint32_t* __restrict__ val2) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n || !flag[j]) return;
  int p = pos[j];
  uint64_t k = key[j];
  int f = (int)(k / (uint64_t)M), l = (int)(k % (uint64_t)M);
  fs_in[p] = (int32_t)val[j];
  fs_fr[p] = f;
  key2[p] = (uint64_t)l * (uint64_t)N + (uint64_t)f;
  val2[p] = (uint32_t)p;
}

// canonical (landmark-major) edge arrays + inverse map frame-sorted → canonical
__global__ void k_gather_edges(int64_t E, const uint64_t* __restrict__ key2,
                               const uint32_t* __restrict__ val2, const int32_t* __restrict__ fs_in,
                               int N, const double* __restrict__ pts, const double* __restrict__ w,
                               int32_t* __restrict__ e_fr, int32_t* __restrict__ e_lm,
                               double* __restrict__ e_pts, double* __restrict__ e_w,
                               int32_t* __restrict__ fr_edge, int32_t* __restrict__ e_in) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= E) return;
  uint64_t k = key2[c];
  int j = (int)val2[c];
  int ein = fs_in[j];
  e_lm[c] = (int)(k / (uint64_t)N);
  e_fr[c] = (int)(k % (uint64_t)N);
  e_pts[3 * c] = pts[3 * (int64_t)ein];
  e_pts[3 * c + 1] = pts[3 * (int64_t)ein + 1];
  e_pts[3 * c + 2] = pts[3 * (int64_t)ein + 2];
  e_w[c] = w ? w[ein] : 1.0;
  e_in[c] = ein;
  fr_edge[j] = (int32_t)c;
}

__global__ void k_histogram(const int32_t* __restrict__ idx, int64_t n, int32_t* __restrict__ cnt) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) atomicAdd(&cnt[idx[j]], 1);
}

// W_k = Σ_{e ∈ track k} w_e, sequential per landmark (deterministic)
__global__ void k_track_weight(int M, const int32_t* __restrict__ off, const double* __restrict__ w,
                               double* __restrict__ W) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  double s = 0.0;
  for (int e = off[k]; e < off[k + 1]; ++e) s += w[e];
  W[k] = s;
}

// ------------------------------------------------ connectivity (min-label + jumping)
__global__ void k_cc_init(int n, int32_t* parent) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) parent[v] = v;
}
__global__ void k_cc_hook(int64_t E, int N, const int32_t* __restrict__ fr,
                          const int32_t* __restrict__ lm, int32_t* parent, int* changed) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  int a = parent[fr[e]], b = parent[N + lm[e]];
  if (a != b) {
    int hi = a > b ? a : b, lo = a > b ? b : a;
    atomicMin(&parent[hi], lo);
    *changed = 1;
  }
}
__global__ void k_cc_jump(int n, int32_t* parent) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int p = parent[v];
  while (p != parent[p]) p = parent[p];
  parent[v] = p;
}
__global__ void k_cc_count(int N, int M, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ lm_off, const int32_t* __restrict__ fr_cnt,
                           int* out) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N + M) return;
  bool present = v < N ? (fr_cnt[v] > 0) : (lm_off[v - N + 1] > lm_off[v - N]);
  if (v < N && fr_cnt[v] == 0) atomicAdd(&out[1], 1);  // unobserved frame
  if (present && parent[v] == v) atomicAdd(&out[0], 1);
}

// ============================================================ H3 S pattern
__global__ void k_pattern_bits(int N, int W32, const int32_t* __restrict__ fr_off,
                               const int32_t* __restrict__ fr_edge, const int32_t* __restrict__ e_lm,
                               const int32_t* __restrict__ lm_off, const int32_t* __restrict__ e_fr,
                               unsigned* __restrict__ bits) {
  int i = blockIdx.x;
  unsigned* row = bits + (int64_t)i * W32;
  if (threadIdx.x == 0) atomicOr(&row[i >> 5], 1u << (i & 31));
  for (int j = fr_off[i]; j < fr_off[i + 1]; ++j) {
    int k = e_lm[fr_edge[j]];
    for (int f = lm_off[k] + threadIdx.x; f < lm_off[k + 1]; f += blockDim.x) {
      int jf = e_fr[f];
      atomicOr(&row[jf >> 5], 1u << (jf & 31));
    }
  }
}
__global__ void k_pattern_count(int N, int W32, const unsigned* __restrict__ bits,
                                int32_t* __restrict__ cnt) {
  int i = blockIdx.x;
  int s = 0;
  for (int w = threadIdx.x; w < W32; w += blockDim.x) s += __popc(bits[(int64_t)i * W32 + w]);
  __shared__ int sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) cnt[i] = sh[0];
}
// one warp per row: enumerate set bits in ascending column order
__global__ void k_pattern_cols(int N, int W32, const unsigned* __restrict__ bits,
                               const int64_t* __restrict__ off, int32_t* __restrict__ colidx,
                               int64_t* __restrict__ rowptr) {
  int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (i >= N) return;
  int64_t base = off[i];  // 64-bit: a near-full pattern has ~N² blocks (> 2³¹ past N ≈ 46 k)
  if (lane == 0) rowptr[i] = base;
  for (int w0 = 0; w0 < W32; w0 += 32) {
    int w = w0 + lane;
    unsigned b = (w < W32) ? bits[(int64_t)i * W32 + w] : 0u;
    int c = __popc(b);
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int64_t pos = base + incl - c;
    while (b) {
      int bit = __ffs(b) - 1;
      colidx[pos++] = w * 32 + bit;
      b &= b - 1;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ============================================================ H4 clique scatter
// CTA i owns: S rows 3i..3i+2 (if i is this rank's frame), C̄ row i−1 (t_i),
// K̄ row i−1.  For each landmark k of frame i (ascending k) the threads update
// H_(i, j_f) for every f in track(k); a __syncthreads between landmarks makes
// the accumulation order fixed.
__global__ void __launch_bounds__(128) k_clique_scatter(
    int N, int f0, int f1, const int32_t* __restrict__ fr_off, const int32_t* __restrict__ fr_edge,
    const int32_t* __restrict__ lm_off, const int32_t* __restrict__ e_fr,
    const double* __restrict__ e_pts, const double* __restrict__ e_w, const double* __restrict__ W,
    const int32_t* __restrict__ e_lm, double* __restrict__ S, int64_t ldq, int row0,
    double* __restrict__ Cb, double* __restrict__ Kb, int64_t ldk) {
  const int i = blockIdx.x;
  const bool own = (i >= f0 && i < f1);
  for (int j = fr_off[i]; j < fr_off[i + 1]; ++j) {
    const int e = fr_edge[j];
    const int k = e_lm[e];
    const double ae0 = e_pts[3 * e], ae1 = e_pts[3 * e + 1], ae2 = e_pts[3 * e + 2];
    const double we = e_w[e];
    const double coef = we / W[k];
    for (int f = lm_off[k] + threadIdx.x; f < lm_off[k + 1]; f += blockDim.x) {
      const int jf = e_fr[f];
      const double af[4] = {e_pts[3 * f], e_pts[3 * f + 1], e_pts[3 * f + 2], 1.0};
      const double ae[4] = {ae0, ae1, ae2, 1.0};
      const double cf = coef * e_w[f];
      double h[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) h[a][b] = -cf * ae[a] * af[b];
      if (f == e) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) h[a][b] += we * ae[a] * ae[b];
      }
      if (own) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double* rowp = S + (int64_t)(3 * i + a - row0) * ldq + 3 * jf;
#pragma unroll
          for (int b = 0; b < 3; ++b) rowp[b] += h[a][b];
        }
      }
      if (i >= 1) {
        double* crow = Cb + (int64_t)(i - 1) * ldq + 3 * jf;
#pragma unroll
        for (int b = 0; b < 3; ++b) crow[b] += h[3][b];
        if (jf >= 1) Kb[(int64_t)(i - 1) * ldk + (jf - 1)] += h[3][3];
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ H4 v2: exact fixed-point
// Row-owned like k_clique_scatter, but the accumulation order no longer
// matters: every term of an output entry is added EXACTLY, as an 88-bit
// fixed-point integer (two signed 44-bit limbs, integer shared-memory
// atomics), and rounded to fp64 once at the end.  So all the (landmark,
// partner) pairs of a frame are processed in parallel (no per-landmark
// barrier chain), every read-modify-write hits shared memory, each output
// entry is written once, and the result is bitwise deterministic (and more
// accurate than any fixed fp64 summation order).  Scale: every term of H
// (App. A) is bounded by T = max_e w_e(1 + |ũ_e|²)
// (|w_e w_f a_e[a] a_f[b]/W_k| ≤ √(w_e w_f)|a_e||a_f|), so with x = term·2^s,
// 2^s·T ≤ 2^70, a sum of up to 2^17 terms stays below 2^87 < 2^88 and each
// limb sum below 2^61; resolution 2^-s ≈ T·2^-70 (≈ 8e-22·T, vs fp64's
// 1.1e-16·T per rounding).
//
// CTA = frame i (row band: S rows 3i..3i+2, C̄ row i−1, K̄ row i−1); output
// columns in chunks of WCF frames.  Per chunk and batch of ≤ SC_THREADS
// landmarks of frame i: (1) one thread per landmark advances its cursor
// through the track (sorted by frame) to the chunk end and caches a_e, w_e,
// w_e/W_k; (2) a block prefix sum flattens the (landmark, partner) pairs;
// (3) one thread per pair adds its ≤ 13 terms.
constexpr int kFxEntries = 13;
template <int WCF, int SC_THREADS>
constexpr size_t scatter_smem() {
  return (size_t)kFxEntries * 2 * WCF * sizeof(long long) +      // accumulators
         (size_t)SC_THREADS * (5 * sizeof(double) + 3 * sizeof(int));  // landmark batch cache
}

template <int WCF>
__device__ __forceinline__ void fx_add(unsigned long long* acc, int entry, int col, double x) {
  // x = term·2^s (|x| < 2^88); two signed limbs of 44 bits, truncated below 2^0
  const double d1 = trunc(x * 0x1p-44);
  const double d0 = trunc(x - d1 * 0x1p44);
  unsigned long long* p = acc + (size_t)entry * 2 * WCF + col;
  atomicAdd(p, (unsigned long long)(long long)d0);
  if (d1 != 0.0) atomicAdd(p + WCF, (unsigned long long)(long long)d1);
}

template <int WCF>
__device__ __forceinline__ double fx_value(const unsigned long long* acc, int entry, int col,
                                           double inv_scale) {
  const unsigned long long* p = acc + (size_t)entry * 2 * WCF + col;
  long long l0 = (long long)p[0], l1 = (long long)p[WCF];
  const long long c = l0 >> 44;  // normalise: l0 ∈ [0, 2^44)
  l0 -= c * (1ll << 44);
  l1 += c;
  return ((double)l1 * 0x1p44 + (double)l0) * inv_scale;
}

// −T per block, T = max_e w_e (1 + |ũ_e|²)  (min-reduced afterwards: max = −min(−·))
__global__ void k_term_bound(int64_t E, const double* __restrict__ pts, const double* __restrict__ w,
                             double* __restrict__ partials) {
  __shared__ double sh[256];
  double m = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double x = pts[3 * e], y = pts[3 * e + 1], z = pts[3 * e + 2];
    m = fmax(m, w[e] * (1.0 + x * x + y * y + z * z));
  }
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = -sh[0];
}

// S_lower: with one rank the SYRK + mirror read only S[3i+a][3j+b] for j ≤ i
template <int WCF, int SC_THREADS>
__global__ void __launch_bounds__(SC_THREADS) k_clique_scatter_fx(
    int N, int f0, int f1, int s_lower_only, const int32_t* __restrict__ fr_off,
    const int32_t* __restrict__ fr_edge, const int32_t* __restrict__ lm_off,
    const int32_t* __restrict__ e_fr, const double* __restrict__ e_pts,
    const double* __restrict__ e_w, const double* __restrict__ W, const int32_t* __restrict__ e_lm,
    double* __restrict__ S, int64_t ldq, int row0, double* __restrict__ Cb,
    double* __restrict__ Kb, int64_t ldk, int32_t* __restrict__ cursor, double scale,
    double inv_scale, int k_only) {
  extern __shared__ unsigned long long acc[];
  double* l_ae = reinterpret_cast<double*>(acc + (size_t)kFxEntries * 2 * WCF);  // [3][T]
  double* l_we = l_ae + 3 * SC_THREADS;
  double* l_coef = l_we + SC_THREADS;
  int* l_p = reinterpret_cast<int*>(l_coef + SC_THREADS);  // first partner in chunk
  int* l_e = l_p + SC_THREADS;                           // the frame's own edge
  int* l_off = l_e + SC_THREADS;                         // exclusive prefix of pair counts
  __shared__ int warp_tot[SC_THREADS / 32];
  __shared__ int batch_pairs;
  const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool own = (i >= f0 && i < f1);
  const int e0 = fr_off[i], nl = fr_off[i + 1] - e0;
  for (int l = tid; l < nl; l += SC_THREADS) cursor[e0 + l] = lm_off[e_lm[fr_edge[e0 + l]]];
  for (int c0 = 0; c0 < N; c0 += WCF) {
    const int c1 = min(N, c0 + WCF);
    const bool needS = !k_only && own && (!s_lower_only || c0 <= i);
    const bool needK = i >= 1 && c0 <= i;
    if (k_only && !needK) break;  // K̄ lower only: no chunk right of the diagonal
    for (int t = tid; t < kFxEntries * 2 * WCF; t += SC_THREADS) acc[t] = 0ull;
    for (int lb = 0; lb < nl; lb += SC_THREADS) {
      // (1) per landmark: partners of this chunk = [p, q) of its frame-sorted track
      const int l = lb + tid;
      int cnt = 0;
      if (l < nl) {
        const int e = fr_edge[e0 + l];
        const int k = e_lm[e];
        const int end = lm_off[k + 1];
        const int p = cursor[e0 + l];
        int q = p;
        while (q < end) {  // 4 independent loads per round
          int v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = (q + u < end) ? e_fr[q + u] : INT32_MAX;
          int adv = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) adv += (v[u] < c1);
          q += adv;
          if (adv < 4) break;
        }
        cursor[e0 + l] = q;
        cnt = q - p;
        l_p[tid] = p;
        l_e[tid] = e;
        l_ae[tid] = e_pts[3 * e];
        l_ae[SC_THREADS + tid] = e_pts[3 * e + 1];
        l_ae[2 * SC_THREADS + tid] = e_pts[3 * e + 2];
        const double we = e_w[e];
        l_we[tid] = we;
        l_coef[tid] = we / W[k];
      }
      // (2) block exclusive scan of the pair counts
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) warp_tot[wid] = x;
      __syncthreads();
      if (wid == 0) {
        int t = lane < SC_THREADS / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, t, o);
          if (lane >= o) t += y;
        }
        if (lane < SC_THREADS / 32) warp_tot[lane] = t;  // inclusive
        if (lane == SC_THREADS / 32 - 1) batch_pairs = t;
      }
      __syncthreads();
      l_off[tid] = x - cnt + (wid > 0 ? warp_tot[wid - 1] : 0);
      __syncthreads();
      // (3) one thread per (landmark, partner) pair
      const int npairs = batch_pairs;
      const int nlb = min(SC_THREADS, nl - lb);
      for (int t = tid; t < npairs; t += SC_THREADS) {
        int lo = 0, hi = nlb - 1;  // last landmark slot with l_off ≤ t
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (l_off[mid] <= t) lo = mid; else hi = mid - 1;
        }
        const int s = lo;
        const int f = l_p[s] + (t - l_off[s]);
        const int jf = e_fr[f];
        const double ae[4] = {l_ae[s], l_ae[SC_THREADS + s], l_ae[2 * SC_THREADS + s], 1.0};
        const double we = l_we[s];
        const double af[4] = {e_pts[3 * f], e_pts[3 * f + 1], e_pts[3 * f + 2], 1.0};
        const double cf = l_coef[s] * e_w[f];
        const int col = jf - c0;
        // h[a][b] = c·a_e[a]·a_f[b], c = −w_e w_f/W_k, or w_e − w_e²/W_k on the
        // diagonal (f = e; exactly 0 for a single-view landmark, W_k = w_e), ×2^s
        const double cp = (f == l_e[s]) ? (we - cf) : -cf;
        if (needS && (!s_lower_only || jf <= i)) {
#pragma unroll
          for (int a2 = 0; a2 < 3; ++a2) {
            const double ca = cp * ae[a2];
#pragma unroll
            for (int b = 0; b < 3; ++b) fx_add<WCF>(acc, 3 * a2 + b, col, ca * af[b] * scale);
          }
        }
        if (i >= 1) {
          if (!k_only) {
#pragma unroll
            for (int b = 0; b < 3; ++b) fx_add<WCF>(acc, 9 + b, col, cp * af[b] * scale);
          }
          if (jf >= 1 && jf <= i) fx_add<WCF>(acc, 12, col, cp * scale);
        }
      }
      __syncthreads();
    }
    // write the chunk: S rows 3i..3i+2 (cols 3c0..), C̄ row i−1, K̄ row i−1 (lower part)
    const int w3 = 3 * (c1 - c0);
    if (needS) {
      const int jmax = s_lower_only ? min(c1, i + 1) : c1;  // frames c0..jmax−1
      const int wS = 3 * (jmax - c0);
      for (int t = tid; t < 3 * wS; t += SC_THREADS) {
        const int a2 = t / wS, x = t % wS, col = x / 3, b = x % 3;
        S[(int64_t)(3 * i + a2 - row0) * ldq + 3 * c0 + x] = fx_value<WCF>(acc, 3 * a2 + b, col, inv_scale);
      }
    }
    if (i >= 1) {
      if (!k_only)
        for (int x = tid; x < w3; x += SC_THREADS)
          Cb[(int64_t)(i - 1) * ldq + 3 * c0 + x] = fx_value<WCF>(acc, 9 + x % 3, x / 3, inv_scale);
      if (needK) {
        const int jlo = max(c0, 1), jhi = min(c1, i + 1);
        for (int j = jlo + tid; j < jhi; j += SC_THREADS)
          Kb[(int64_t)(i - 1) * ldk + (j - 1)] = fx_value<WCF>(acc, 12, j - c0, inv_scale);
      }
    }
    __syncthreads();
  }
}

// ============================================================ dense fp64 kernels
// The O(N³) updates are the DMMA kernel of dgemm_tn.cu (TN shape, see there).

// ---------------------------------------------------------------- Cholesky
constexpr int NB = 64;

__global__ void k_zero_upper(double* A, int m, int64_t lda) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)m * m) return;
  int i = (int)(t / m), j = (int)(t % m);
  if (j > i) A[(int64_t)i * lda + j] = 0.0;
}

// max_i A[i][i] (one block; used to make the Cholesky pivot test relative)
__global__ void k_diag_max(const double* __restrict__ A, int m, int64_t lda, double* out) {
  __shared__ double sh[256];
  double v = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) v = fmax(v, A[(int64_t)i * lda + i]);
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// One panel step of the blocked Cholesky, fused: every CTA factors the
// nb×nb diagonal block in shared memory (redundantly — it is ≈ 3 µs of work
// and saves a dependent launch; CTA 0 stores it in a side slot that
// k_chol_diag_back copies into place after the last step), then each thread
// solves one row of the panel below, x·L11ᵀ = a  (row in registers).
// Diagonal-block factorisation: 16×16 threads, thread (ti, tl) owns the 4×4
// sub-block rows 4ti.., columns 4tl.. of the trailing update (no index
// division in the inner loop).
template <int NBT>
__global__ void __launch_bounds__(256) k_chol_panel(double* __restrict__ Akk, int64_t lda, int nb,
                                                    int rows, double rel_tol,
                                                    const double* __restrict__ scale,
                                                    int* __restrict__ err,
                                                    double* __restrict__ L11_out,
                                                    double* __restrict__ Ut, int64_t ldu) {
  static_assert(NBT == 64, "16 x 16 threads x 4 x 4");
  __shared__ double a[NBT][NBT + 1];
  const double pivot_tol = rel_tol * (*scale);
  const int tid = threadIdx.x, ti = tid >> 4, tl = tid & 15;
  for (int t = tid; t < NBT * NBT; t += 256) {
    const int i = t >> 6, j = t & 63;
    a[i][j] = (i < nb && j < nb && j <= i) ? Akk[(int64_t)i * lda + j] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  // Right-looking factorisation with ONE barrier per column: every thread
  // derives 1/√d_j itself, updates its 4×4 sub-block with the unscaled column
  // (a_il −= (a_ij·s)(a_lj·s), s = 1/√d_j), and scales its part of column j
  // one step later (column j is no longer read by then).
  double inv_prev = 1.0, sq_prev = 1.0;
  for (int j = 0; j < nb; ++j) {
    if (j > 0 && tl == (j - 1) >> 2) {  // finish column j−1 (and its diagonal)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int i = 4 * ti + x;
        if (i > j - 1 && i < nb) a[i][j - 1] *= inv_prev;
      }
      if (ti == (j - 1) >> 2) a[j - 1][j - 1] = sq_prev;
    }
    double d = a[j][j];
    if (!(d > pivot_tol)) {
      if (tid == 0 && blockIdx.x == 0) atomicOr(err, 1);
      d = 1.0;
    }
    const double sq = sqrt(d);
    const double inv = 1.0 / sq;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int i = 4 * ti + x;
      if (i > j && i < nb) {
        const double lij = a[i][j] * inv;
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int l = 4 * tl + y;
          if (l > j && l <= i) a[i][l] = fma(-lij, a[l][j] * inv, a[i][l]);
        }
      }
    }
    inv_prev = inv;
    sq_prev = sq;
    __syncthreads();
  }
  if (nb > 0 && tl == (nb - 1) >> 2) {  // last column: only its diagonal
    if (ti == (nb - 1) >> 2) a[nb - 1][nb - 1] = sq_prev;
  }
  __syncthreads();
  if (blockIdx.x == 0)  // into a side slot: other CTAs may still be reading Akk
    for (int t = tid; t < NBT * NBT; t += 256) L11_out[t] = a[t >> 6][t & 63];
  __shared__ double rdiag[NBT];  // 1/L_jj: the row solve multiplies (no fp64 division chain)
  if (tid < NBT) rdiag[tid] = 1.0 / a[tid][tid];
  __syncthreads();
  // panel rows: X·L11ᵀ = A21
  const int r = blockIdx.x * 256 + tid;
  if (r >= rows) return;
  double* row = Akk + (int64_t)(nb + r) * lda;
  double x[NBT];
#pragma unroll
  for (int j = 0; j < NBT; ++j) x[j] = (j < nb) ? row[j] : 0.0;  // all loads in flight at once
#pragma unroll
  for (int j = 0; j < NBT; ++j) {
    if (j < nb) {
      double s2 = x[j];
#pragma unroll
      for (int q = 0; q < j; ++q) s2 = fma(-x[q], a[j][q], s2);
      x[j] = s2 * rdiag[j];
    }
  }
#pragma unroll
  for (int j = 0; j < NBT; ++j)
    if (j < nb) {
      row[j] = x[j];
      Ut[(int64_t)j * ldu + r] = x[j];  // the same panel transposed (U = Lᵀ rows), coalesced in r
    }
}

// L11 slots → diagonal blocks (strict upper part of each block zeroed)
__global__ void k_chol_diag_back(const double* __restrict__ slots, double* __restrict__ A,
                                 int64_t lda, int m) {
  const int blk = blockIdx.x, kb = blk * NB, nb = min(NB, m - kb);
  const double* sl = slots + (size_t)blk * NB * NB;
  for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
    const int i = t / NB, j = t % NB;
    if (i < nb && j < nb) A[(int64_t)(kb + i) * lda + kb + j] = (j <= i) ? sl[t] : 0.0;
  }
}

// Blocked right-looking Cholesky A = LLᵀ (lower, row-major, in place).  Each
// panel step also writes the panel transposed — the rows kb..kb+nb of U = Lᵀ
// right of the diagonal block — into U (if given; else into a one-panel
// scratch), so the trailing update A₂₂ −= L₂₁L₂₁ᵀ is the TN DMMA kernel on
// lower tiles, and a later TRSM can use U as its TN operand too.
bool dense_cholesky(xm_ctx* c, double* A, int m, int64_t lda, double rel_tol, bool throw_on_fail,
                    double* U, int64_t ldu) {
  if (m <= 0) return true;
  c->flags.alloc(16);
  c->scal.alloc(64);
  XM_CUDA(cudaMemsetAsync(c->flags.p, 0, sizeof(int), c->stream));
  double* d_scale = c->scal.p + 63;
  k_diag_max<<<1, 256, 0, c->stream>>>(A, m, lda, d_scale);
  XM_CHECK_LAUNCH();
  count_launch(c);
  DBuf<double>& slots = scratch_f64(c, "chol_l11");
  slots.alloc((size_t)ceil_div(m, NB) * NB * NB);
  DBuf<double>& panel = scratch_f64(c, "chol_panel");
  if (!U) {
    ldu = round_up(std::max(m, 1), 32);
    panel.alloc((size_t)NB * ldu);
  }
  // Look-ahead: the trailing update of panel k is split into (a) the next
  // panel's 64 columns (all rows below) on the main stream, and (b) the rest on
  // a side stream, so the latency-bound factorisation of panel k+1 runs
  // concurrently with the big update (b) of panel k.  (a) of panel k+1 waits
  // for (b) of panel k (both write the columns of panel k+2).  Without a U
  // buffer (the scratch panel is reused every step) the plain order is kept.
  const bool look = U != nullptr && c->cap_target == nullptr && !std::getenv("XM_NO_CHOL_LOOKAHEAD");
  if (look && !c->aux_stream) {
    XM_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
    XM_CUDA(cudaEventCreateWithFlags(&c->ev_la, cudaEventDisableTiming));
    XM_CUDA(cudaEventCreateWithFlags(&c->ev_lb, cudaEventDisableTiming));
  }
  bool pending_b = false;
  for (int kb = 0; kb < m; kb += NB) {
    int nb = std::min(NB, m - kb);
    double* Akk = A + (int64_t)kb * lda + kb;
    int rows = m - kb - nb;
    // U panel: rows kb.., columns kb+nb.. (scratch: rows 0.., columns 0..)
    double* Up = U ? U + (int64_t)kb * ldu + (kb + nb) : panel.p;
    k_chol_panel<NB><<<std::max(1, ceil_div(rows, 256)), 256, 0, c->stream>>>(
        Akk, lda, nb, rows, rel_tol, d_scale, c->flags.p, slots.p + (size_t)(kb / NB) * NB * NB,
        Up, ldu);
    XM_CHECK_LAUNCH();
    count_launch(c);
    if (rows <= 0) continue;
    double* A22 = A + (int64_t)(kb + nb) * lda + (kb + nb);
    if (!look) {
      dgemm_tn(c, true, rows, rows, nb, -1.0, Up, ldu, Up, ldu, 1.0, A22, lda);
      continue;
    }
    const int nb2 = std::min(NB, rows);
    if (pending_b) XM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_lb, 0));  // (b) of panel k−1
    // (a) the next panel's columns, every row below (its diagonal block's upper part
    // is scratch: k_chol_panel reads the lower part, k_chol_diag_back rewrites it)
    dgemm_tn(c, false, rows, nb2, nb, -1.0, Up, ldu, Up, ldu, 1.0, A22, lda);
    pending_b = false;
    if (rows > nb2) {
      XM_CUDA(cudaEventRecord(c->ev_la, c->stream));
      XM_CUDA(cudaStreamWaitEvent(c->aux_stream, c->ev_la, 0));
      cudaStream_t main = c->stream;
      c->stream = c->aux_stream;  // (b) the rest of the trailing matrix, lower tiles
      try {
        dgemm_tn(c, true, rows - nb2, rows - nb2, nb, -1.0, Up + nb2, ldu, Up + nb2, ldu, 1.0,
                 A22 + (int64_t)nb2 * lda + nb2, lda);
      } catch (...) {
        c->stream = main;
        throw;
      }
      c->stream = main;
      XM_CUDA(cudaEventRecord(c->ev_lb, c->aux_stream));
      pending_b = true;
    }
  }
  if (pending_b) XM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_lb, 0));
  k_chol_diag_back<<<ceil_div(m, NB), 256, 0, c->stream>>>(slots.p, A, lda, m);
  XM_CHECK_LAUNCH();
  count_launch(c);
  if (throw_on_fail) {
    k_zero_upper<<<ceil_div((int64_t)m * m, 256), 256, 0, c->stream>>>(A, m, lda);
    XM_CHECK_LAUNCH();
    count_launch(c);
  }
  int h_err = 0;
  XM_CUDA(cudaMemcpyAsync(&h_err, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (h_err && throw_on_fail)
    throw Error(XM_EDISCONNECTED, "graph numerically disconnected (Cholesky pivot)");
  return h_err == 0;
}

// Z + εI with Z = Q − blkdiag(Λ) (Eq. (16)); lower triangle incl. diagonal is all potrf reads.
__global__ void k_form_z_shift(const double* __restrict__ Q, int64_t ldq, int n,
                               const double* __restrict__ lam, double eps, double* __restrict__ Z,
                               const double* __restrict__ regd) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * n) return;
  int i = (int)(t / n), j = (int)(t % n);
  if (j > i) return;
  double v = Q[(int64_t)i * ldq + j];
  if (i / 3 == j / 3) {
    const double* L = lam + 6 * (i / 3);
    int a = i % 3, b = j % 3;
    const int idx[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
    v -= L[idx[a][b]];
    if (i == j) v += eps + (regd ? regd[i / 3] : 0.0);  // Z_λ = Q + blkdiag(d I) − blkdiag(Λ)
  }
  Z[(int64_t)i * ldq + j] = v;
}

// tr(A) and ‖A‖_F² of a symmetric A from its lower triangle (one block, fixed order)
__global__ void k_sym_stats(const double* __restrict__ A, int64_t lda, int n, double* out) {
  __shared__ double st[256], sf[256];
  double tr = 0.0, fr = 0.0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const double* row = A + (int64_t)i * lda;
    for (int j = threadIdx.x; j <= i; j += blockDim.x) {
      const double v = row[j];
      fr = fma(j == i ? 1.0 : 2.0, v * v, fr);
      if (j == i) tr += v;
    }
  }
  st[threadIdx.x] = tr;
  sf[threadIdx.x] = fr;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      st[threadIdx.x] += st[threadIdx.x + s];
      sf[threadIdx.x] += sf[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = st[0];
    out[2 * blockIdx.x + 1] = sf[0];
  }
}

// PSD test of Z(y) (Alg. 1): Cholesky of Z + sI runs to completion ⇔
// (in exact arithmetic) λ_min(Z) > −s.  In floating point, completion means
// Z̃ + sI + ΔA = L̂L̂ᵀ with |ΔA| ≤ γ_{n+1}|L̂||L̂ᵀ| (Cholesky backward error,
// any summation order), and ‖|L̂||L̂ᵀ|‖₂ ≤ ‖L̂‖_F² = tr(L̂L̂ᵀ) ≈ tr(Z + sI); Z̃ =
// fl(Q − Λ) differs from Z by ≤ u|Z|.  So success certifies
//   λ_min(Z) ≥ −s − γ_{n+1}·tr(Z + sI)·(1 + 2γ_{n+1}) − u‖Z‖_F   (= *lower).
// Single-rank Q only.  Zw ← L (lower), U ← Lᵀ if `U` is given.
bool psd_test_cholesky(xm_ctx* c, double s, double* lower, double* U, int64_t ldu) {
  if (c->world != 1) throw Error(XM_EINVAL, "Cholesky PSD test needs the full Q on one rank");
  const int n = c->n;
  c->Zw.alloc((size_t)n * c->ldq);
  k_form_z_shift<<<ceil_div((int64_t)n * n, 256), 256, 0, c->stream>>>(
      c->Q.p, c->ldq, n, c->lam.p, s, c->Zw.p, c->opt.scale_reg != 0.0 ? c->regd.p : nullptr);
  XM_CHECK_LAUNCH();
  count_launch(c);
  DBuf<double>& sp = scratch_f64(c, "zstats");
  constexpr int kSB = 148;
  sp.alloc(2 * kSB);
  k_sym_stats<<<kSB, 256, 0, c->stream>>>(c->Zw.p, c->ldq, n, sp.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  std::vector<double> hs(2 * kSB);
  XM_CUDA(cudaMemcpyAsync(hs.data(), sp.p, 2 * kSB * 8, cudaMemcpyDeviceToHost, c->stream));
  const bool ok = dense_cholesky(c, c->Zw.p, n, c->ldq, 0.0, false, U, ldu);  // syncs
  double tr = 0.0, fr2 = 0.0;
  for (int b = 0; b < kSB; ++b) {
    tr += hs[2 * b];
    fr2 += hs[2 * b + 1];
  }
  const double u = 1.1102230246251565e-16;
  const double g = (n + 1) * u / (1.0 - (n + 1) * u);
  if (lower) *lower = -s - g * std::fabs(tr) * (1.0 + 2.0 * g) - u * std::sqrt(fr2);
  return ok;
}

// Forward substitution of a diagonal block for many right-hand sides:
// B[0:nb, :] ← L11⁻¹ B[0:nb, :] (one thread per column; L11 in smem).
template <int NBT>
__global__ void __launch_bounds__(128) k_trsm_block_cols(const double* __restrict__ L11,
                                                         int64_t ldl, double* __restrict__ B,
                                                         int64_t ldb, int nb, int ncols) {
  __shared__ double l[NBT][NBT + 1];
  for (int t = threadIdx.x; t < nb * nb; t += blockDim.x) {
    int i = t / nb, j = t % nb;
    l[i][j] = (j <= i) ? L11[(int64_t)i * ldl + j] : 0.0;
  }
  __syncthreads();
  int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double x[NBT];
#pragma unroll
  for (int j = 0; j < NBT; ++j) x[j] = (j < nb) ? B[(int64_t)j * ldb + col] : 0.0;
#pragma unroll
  for (int j = 0; j < NBT; ++j) {
    if (j < nb) {
      double s = x[j];
#pragma unroll
      for (int q = 0; q < j; ++q) s -= l[j][q] * x[q];
      x[j] = s / l[j][j];
    }
  }
#pragma unroll
  for (int j = 0; j < NBT; ++j)
    if (j < nb) B[(int64_t)j * ldb + col] = x[j];
}

__global__ void k_set_diag(double* A, int n, int64_t lda) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[(int64_t)i * lda + i] = 1.0;
}

__global__ void k_eye(double* T, int m, int64_t ld) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * m) return;
  const int i = t / m, j = t % m;
  T[(int64_t)i * ld + j] = (i == j) ? 1.0 : 0.0;
}

void identity(xm_ctx* c, double* A, int n, int64_t lda) {
  XM_CUDA(cudaMemsetAsync(A, 0, (size_t)n * lda * sizeof(double), c->stream));
  k_set_diag<<<ceil_div(n, 256), 256, 0, c->stream>>>(A, n, lda);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

__global__ void k_transpose(const double* __restrict__ S, int64_t lds, double* __restrict__ D,
                            int64_t ldd, int rows, int cols) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = by + y, cc = bx + threadIdx.x;
    tile[y][threadIdx.x] = (r < rows && cc < cols) ? S[(int64_t)r * lds + cc] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = bx + y, cc = by + threadIdx.x;  // D[cc_src][r_src]
    if (r < cols && cc < rows) D[(int64_t)r * ldd + cc] = tile[threadIdx.x][y];
  }
}

// Rows [k0, k1) of B ← L⁻¹ B restricted to the diagonal block L[k0:k1, k0:k1]
// (64-row diagonal solves with their short TN updates inside the block).
static void trsm_block_inner(xm_ctx* c, const double* L, int64_t ldl, const double* U, int64_t ldu,
                             int k0, int k1, double* B, int ncols, int64_t ldb) {
  for (int kb = k0; kb < k1; kb += NB) {
    int nb = std::min(NB, k1 - kb);
    const double* Lkk = L + (int64_t)kb * ldl + kb;
    double* Bk = B + (int64_t)(kb - k0) * ldb;
    k_trsm_block_cols<NB><<<ceil_div(ncols, 128), 128, 0, c->stream>>>(Lkk, ldl, Bk, ldb, nb, ncols);
    XM_CHECK_LAUNCH();
    count_launch(c);
    int rows = k1 - kb - nb;
    if (rows > 0)
      dgemm_tn(c, false, rows, ncols, nb, -1.0, U + (int64_t)kb * ldu + (kb + nb), ldu, Bk, ldb, 1.0,
               B + (int64_t)(kb + nb - k0) * ldb, ldb);
  }
}

// B ← L⁻¹B (L lower m×m).  Super-blocks of SB = 512 rows: the diagonal block's
// inverse L_ss⁻¹ (SB × SB, from the 64-row solves on an identity) is applied
// as ONE TN DMMA product (B_s ← L_ss⁻¹ B_s, via a scratch row block), then the
// rows below get ONE TN DMMA update with K = SB (U = Lᵀ from the
// factorisation is the A operand: L₂₁[i][k] = U[k][i]).  The serial 64-row
// solves only ever touch SB columns.
// lower_rhs: B is lower triangular (B[i][j] = 0 for j > i, e.g. the identity
// when inverting L) — then so is the solution, and super-block rows sb..se only
// carry columns < se: m³/3 instead of m³ flops.
// The super-block inverses do not depend on B: they are all computed first,
// round-robin on kTrsmStreams forked streams (each chain — 8 serial 64-row
// solves of 4 CTAs and their small updates — is latency-bound, E: ≈ 1.4 ms per
// super-block, 29 ms in series), then B's super-block chain runs on the main
// stream.  Same kernels, same arithmetic (bitwise identical); XM_NO_TRSM_FORK=1:
// in series on the main stream.
static void trsm_superblock_inverse(xm_ctx* c, const double* L, int64_t ldl, const double* U,
                                    int64_t ldu, int sb, int se, double* T, double* Tt, int SB) {
  const int s = se - sb;
  k_eye<<<ceil_div(s * s, 256), 256, 0, c->stream>>>(T, s, SB);
  XM_CHECK_LAUNCH();
  trsm_block_inner(c, L, ldl, U, ldu, sb, se, T, s, SB);  // T = L_ss⁻¹
  k_transpose<<<dim3(ceil_div(s, 32), ceil_div(s, 32)), dim3(32, 8), 0, c->stream>>>(T, SB, Tt, SB, s, s);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
}

void dense_trsm_lower_left(xm_ctx* c, const double* L, int m, int64_t ldl, const double* U,
                           int64_t ldu, double* B, int ncols, int64_t ldb, bool lower_rhs) {
  const int SB = c->trsm_sb;
  const int nsb = ceil_div(m, SB);
  static const bool no_fork = std::getenv("XM_NO_TRSM_FORK") != nullptr;
  const bool fork = !no_fork && nsb > 1 && c->cap_target == nullptr;  // not inside a graph capture
  constexpr int kS = xm_ctx::kTrsmStreams;
  DBuf<double>& T = scratch_f64(c, "trsm_inv");
  DBuf<double>& Tt = scratch_f64(c, "trsm_invT");
  DBuf<double>& X = scratch_f64(c, "trsm_rows");
  T.alloc((size_t)(fork ? kS : 1) * SB * SB);         // one per stream
  Tt.alloc((size_t)(fork ? nsb : 1) * SB * SB);       // every super-block's L_ss⁻ᵀ
  X.alloc((size_t)SB * ldb);
  if (fork) {
    for (int q = 0; q < kS; ++q)
      if (!c->trsm_streams[q]) XM_CUDA(cudaStreamCreateWithFlags(&c->trsm_streams[q], cudaStreamNonBlocking));
    for (int q = 0; q <= kS; ++q)
      if (!c->trsm_ev[q]) XM_CUDA(cudaEventCreateWithFlags(&c->trsm_ev[q], cudaEventDisableTiming));
    XM_CUDA(cudaEventRecord(c->trsm_ev[kS], c->stream));
    const cudaStream_t main = c->stream;
    for (int q = 0; q < kS; ++q) XM_CUDA(cudaStreamWaitEvent(c->trsm_streams[q], c->trsm_ev[kS], 0));
    try {
      for (int b = 0; b < nsb; ++b) {
        c->stream = c->trsm_streams[b % kS];
        trsm_superblock_inverse(c, L, ldl, U, ldu, b * SB, std::min(m, (b + 1) * SB),
                                T.p + (size_t)(b % kS) * SB * SB, Tt.p + (size_t)b * SB * SB, SB);
      }
    } catch (...) {
      c->stream = main;
      throw;
    }
    c->stream = main;
    for (int q = 0; q < kS; ++q) {
      XM_CUDA(cudaEventRecord(c->trsm_ev[q], c->trsm_streams[q]));
      XM_CUDA(cudaStreamWaitEvent(c->stream, c->trsm_ev[q], 0));
    }
  }
  for (int sb = 0; sb < m; sb += SB) {
    const int se = std::min(m, sb + SB), s = se - sb;
    const double* Ts = Tt.p + (fork ? (size_t)(sb / SB) * SB * SB : 0);
    if (!fork) trsm_superblock_inverse(c, L, ldl, U, ldu, sb, se, T.p, Tt.p, SB);
    const int nc = lower_rhs ? std::min(ncols, se) : ncols;  // columns ≥ se of rows < se are 0
    // X = L_ss⁻¹ B_s :  X[i][j] = Σ_k Tt[k][i] B[sb + k][j]
    dgemm_tn(c, false, s, nc, s, 1.0, Ts, SB, B + (int64_t)sb * ldb, ldb, 0.0, X.p, ldb);
    XM_CUDA(cudaMemcpy2DAsync(B + (int64_t)sb * ldb, ldb * sizeof(double), X.p, ldb * sizeof(double),
                              (size_t)nc * sizeof(double), s, cudaMemcpyDeviceToDevice, c->stream));
    if (se < m)
      dgemm_tn(c, false, m - se, nc, s, -1.0, U + (int64_t)sb * ldu + se, ldu,
               B + (int64_t)sb * ldb, ldb, 1.0, B + (int64_t)se * ldb, ldb);
  }
}

// out[k][j] = B[k][j] for j < wv, 0 for wv ≤ j < w (k < m): a column slice packed
// contiguous for the all-gather of the column-sharded TRSM
__global__ void k_pack_block(int m, int w, int wv, const double* __restrict__ B, int64_t ldb,
                             double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)m * w) return;
  const int64_t k = t / w;
  const int j = (int)(t - k * w);
  out[t] = (j < wv) ? B[k * ldb + j] : 0.0;
}

// Q[i][j] (j > i) ← Q[j][i]: exact symmetry after a lower-triangle SYRK.
__global__ void k_mirror(double* Q, int n, int64_t ldq) {
  __shared__ double tile[32][33];
  int bi = blockIdx.y, bj = blockIdx.x;  // destination tile (bi row, bj col), bj > bi
  if (bj < bi) return;
  int tx = threadIdx.x, ty = threadIdx.y;
  // read source tile (rows bj*32.., cols bi*32..) — lower part
  for (int y = ty; y < 32; y += blockDim.y) {
    int r = bj * 32 + y, cc = bi * 32 + tx;
    tile[y][tx] = (r < n && cc < n) ? Q[(int64_t)r * ldq + cc] : 0.0;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += blockDim.y) {
    int r = bi * 32 + y, cc = bj * 32 + tx;
    if (r < n && cc < n && cc > r) Q[(int64_t)r * ldq + cc] = tile[tx][y];
  }
}

void mirror_lower(xm_ctx* c, double* Q, int n, int64_t ldq) {
  dim3 grid(ceil_div(n, 32), ceil_div(n, 32));
  k_mirror<<<grid, dim3(32, 8), 0, c->stream>>>(Q, n, ldq);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

// Σ Q_ij² over this rank's rows; band layout (row0 ≥ 0): only the lower
// trapezoid is stored, so Σ = Σ_{j<i} 2Q_ij² + Σ_{j=i} Q_ii² over global rows i.
// Rows are distributed over the blocks, columns over the threads (coalesced,
// no per-element index division).
__global__ void k_sumsq_rows(const double* __restrict__ Q, int rows, int n, int64_t ldq,
                             double* __restrict__ partials, int row0) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = blockIdx.x; i < rows; i += gridDim.x) {
    const double* q = Q + (int64_t)i * ldq;
    const int gi = row0 + i;
    const int jend = (row0 >= 0) ? min(n, gi + 1) : n;
    for (int j = threadIdx.x; j < jend; j += blockDim.x) {
      double v = q[j];
      if (row0 >= 0 && j < gi) v *= 1.4142135623730951;
      acc = fma(v, v, acc);
    }
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

// The matrix-free mode's per-product time model (one rank): 1/world of each
// mode's algorithmic bytes at its measured rate — the dense lower-triangle
// stream at ≈ 6.1 TB/s plus one all-reduce, the matrix-free product at
// ≈ 2.85 TB/s plus five dependent launches and five all-reduces (≈ 20 µs each
// assumed over NVLink) — and the dense layout must fit (Q rows, G, K̄ factor).
// E: matrix-free on 1–2 GPUs, the dense band at 4–8; A–D: dense.
bool prefer_implicit(int N, int64_t E, int world) {
  const double n = 3.0 * N, m = N - 1.0, P = world, ar = 20e-6;
  const double t_dense = 8.0 * n * (n + 1.0) / 2.0 / P / 6.1e12 + (world > 1 ? ar : 0.0);
  const double t_imp = (80.0 * (double)E + 8.0 * m * (m + 1.0) / 2.0) / P / 2.85e12 + 15e-6 +
                       (world > 1 ? 5.0 * ar : 0.0);
  const double dense_bytes = 8.0 * n * n / P + 8.0 * m * n + 3.0 * 8.0 * m * m;  // Q rows, G, K̄ (+L, U)
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && dense_bytes > 0.9 * (double)total_b) return true;
  return t_imp < t_dense;
}

// H3: the co-visibility BSR pattern of S (bitmap per row → counts → 64-bit
// row offsets (host prefix sum) → sorted column lists)
void build_s_pattern(xm_ctx* c, int N) {
  int W32 = ceil_div(N, 32);
  DBuf<uint32_t>& bits = scratch_u32(c, "pattern_bits");
  bits.alloc((size_t)N * W32);
  XM_CUDA(cudaMemsetAsync(bits.p, 0, (size_t)N * W32 * 4, c->stream));
  k_pattern_bits<<<N, 128, 0, c->stream>>>(N, W32, c->fr_off.p, c->fr_edge.p, c->e_lm.p,
                                           c->lm_off.p, c->e_fr.p, bits.p);
  XM_CHECK_LAUNCH();
  DBuf<int32_t>& rc = scratch_i32(c, "pattern_rc");
  DBuf<int64_t>& ro = scratch_i64(c, "pattern_ro");
  rc.alloc(N);
  ro.alloc(N + 1);
  k_pattern_count<<<N, 256, 0, c->stream>>>(N, W32, bits.p, rc.p);
  XM_CHECK_LAUNCH();
  std::vector<int32_t> cnt(N);
  std::vector<int64_t> off(N + 1, 0);
  XM_CUDA(cudaMemcpyAsync(cnt.data(), rc.p, (size_t)N * 4, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  for (int i = 0; i < N; ++i) off[i + 1] = off[i] + cnt[i];
  const int64_t nnzb = off[N];
  XM_CUDA(cudaMemcpyAsync(ro.p, off.data(), (size_t)(N + 1) * 8, cudaMemcpyHostToDevice, c->stream));
  c->nnzb = nnzb;
  c->stats.nnzb_S = nnzb;
  c->s_rowptr.alloc(N + 1);
  c->s_colidx.alloc((size_t)std::max<int64_t>(nnzb, 1));
  k_pattern_cols<<<ceil_div(N, 8), 256, 0, c->stream>>>(N, W32, bits.p, ro.p, c->s_colidx.p,
                                                       c->s_rowptr.p);
  XM_CHECK_LAUNCH();
  XM_CUDA(cudaMemcpyAsync(c->s_rowptr.p + N, ro.p + N, 8, cudaMemcpyDeviceToDevice, c->stream));
  count_launch(c, 3);
  sync(c);
  bits.release();
  c->pattern_valid = true;
}

// ============================================================ driver
void build_Q_device(xm_ctx* c, int N, int M, int64_t E, const int32_t* fr_in, const int32_t* lm_in,
                    const double* pts_in, const double* w_in) {
  if (N < 1 || M < 1 || E < 1) throw Error(XM_EINVAL, "empty view graph");
  if (E >= (int64_t)INT32_MAX) throw Error(XM_EINVAL, "too many observations");
  const int T = 256;
  const bool verbose = std::getenv("XM_VERBOSE") != nullptr;
  double tph = 0.0;
  NvtxRange nvtx_all("build_Q");
  auto phase = [&](const char* nm) {
    nvtxMarkA(nm);
    if (!verbose) return;
    sync(c);
    double t = std::chrono::duration<double, std::milli>(
                   std::chrono::steady_clock::now().time_since_epoch()).count();
    if (tph > 0.0) fprintf(stderr, "[xm build] %-14s %9.3f ms\n", nm, t - tph);
    tph = t;
  };
  phase("start");
  // stage inputs on the device
  DBuf<int32_t>& d_fr = scratch_i32(c, "in_fr");
  DBuf<int32_t>& d_lm = scratch_i32(c, "in_lm");
  DBuf<double>& d_pts = scratch_f64(c, "in_pts");
  DBuf<double>& d_w = scratch_f64(c, "in_w");
  const int32_t* fr = fr_in;
  const int32_t* lm = lm_in;
  const double* pts = pts_in;
  const double* w = w_in;
  if (!is_device_ptr(fr_in)) { d_fr.alloc(E); copy_in(c, d_fr.p, fr_in, E * 4); fr = d_fr.p; }
  if (!is_device_ptr(lm_in)) { d_lm.alloc(E); copy_in(c, d_lm.p, lm_in, E * 4); lm = d_lm.p; }
  if (!is_device_ptr(pts_in)) { d_pts.alloc(3 * E); copy_in(c, d_pts.p, pts_in, E * 24); pts = d_pts.p; }
  if (w_in && !is_device_ptr(w_in)) { d_w.alloc(E); copy_in(c, d_w.p, w_in, E * 8); w = d_w.p; }

  c->flags.alloc(16);
  XM_CUDA(cudaMemsetAsync(c->flags.p, 0, 16 * sizeof(int), c->stream));
  // ---- H1: validate, key = (frame, landmark)
  DBuf<uint64_t>& key = scratch_u64(c, "key");
  DBuf<uint64_t>& key2 = scratch_u64(c, "key2");
  DBuf<uint64_t>& tk = scratch_u64(c, "sort_tk");
  DBuf<uint32_t>& val = scratch_u32(c, "val");
  DBuf<uint32_t>& val2 = scratch_u32(c, "val2");
  DBuf<uint32_t>& tv = scratch_u32(c, "sort_tv");
  key.alloc(E);
  val.alloc(E);
  k_validate<<<ceil_div(E, T), T, 0, c->stream>>>(E, N, M, fr, lm, pts, w, c->flags.p, key.p, val.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  int h_err = 0;
  XM_CUDA(cudaMemcpyAsync(&h_err, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (h_err & ERR_RANGE) throw Error(XM_EINVAL, "index out of range");
  if (h_err & ERR_WEIGHT) throw Error(XM_EINVAL, "non-positive or non-finite weight");
  if (h_err & ERR_POINT) throw Error(XM_EINVAL, "non-finite point or non-positive depth");
  int bits_fl = 1;
  while (bits_fl < 64 && ((uint64_t)N * (uint64_t)M) > (1ull << bits_fl)) ++bits_fl;
  radix_sort_u64(c, key.p, val.p, E, bits_fl, tk, tv);
  phase("validate+sort1");
  // ---- dedupe (stable sort ⇒ the first occurrence of a key is the earliest input)
  DBuf<int32_t>& flag = scratch_i32(c, "flag");
  DBuf<int32_t>& pos = scratch_i32(c, "pos");
  flag.alloc(E);
  pos.alloc(E);
  k_first_flags<<<ceil_div(E, T), T, 0, c->stream>>>(key.p, E, flag.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  int32_t* d_total = c->flags.p + 4;
  exclusive_scan_i32(c, flag.p, pos.p, E, d_total);
  int32_t Ek = 0;
  XM_CUDA(cudaMemcpyAsync(&Ek, d_total, 4, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  c->stats.n_dup = E - Ek;
  c->E = Ek;
  DBuf<int32_t>& fs_in = scratch_i32(c, "fs_in");
  DBuf<int32_t>& fs_fr = scratch_i32(c, "fs_fr");
  fs_in.alloc(Ek);
  fs_fr.alloc(Ek);
  key2.alloc(Ek);
  val2.alloc(Ek);
  k_compact_fs<<<ceil_div(E, T), T, 0, c->stream>>>(key.p, val.p, flag.p, pos.p, E, M, N, fs_in.p,
                                                   fs_fr.p, key2.p, val2.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  phase("dedupe");
  // ---- H2: canonical (landmark, frame) order
  radix_sort_u64(c, key2.p, val2.p, Ek, bits_fl, tk, tv);
  c->e_fr.alloc(Ek);
  c->e_lm.alloc(Ek);
  c->e_pts.alloc(3 * Ek);
  c->e_w.alloc(Ek);
  c->fr_edge.alloc(Ek);
  c->e_in.alloc(Ek);
  k_gather_edges<<<ceil_div(Ek, T), T, 0, c->stream>>>(Ek, key2.p, val2.p, fs_in.p, N, pts, w,
                                                      c->e_fr.p, c->e_lm.p, c->e_pts.p, c->e_w.p,
                                                      c->fr_edge.p, c->e_in.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  DBuf<int32_t>& cnt = scratch_i32(c, "cnt");
  cnt.alloc((size_t)std::max(N, M) + 1);
  c->lm_off.alloc(M + 1);
  c->fr_off.alloc(N + 1);
  XM_CUDA(cudaMemsetAsync(cnt.p, 0, (M + 1) * 4, c->stream));
  k_histogram<<<ceil_div(Ek, T), T, 0, c->stream>>>(c->e_lm.p, Ek, cnt.p);
  XM_CHECK_LAUNCH();
  exclusive_scan_i32(c, cnt.p, c->lm_off.p, M + 1, nullptr);
  DBuf<int32_t>& fcnt = scratch_i32(c, "fcnt");
  fcnt.alloc(N + 1);
  XM_CUDA(cudaMemsetAsync(fcnt.p, 0, (N + 1) * 4, c->stream));
  k_histogram<<<ceil_div(Ek, T), T, 0, c->stream>>>(fs_fr.p, Ek, fcnt.p);
  XM_CHECK_LAUNCH();
  exclusive_scan_i32(c, fcnt.p, c->fr_off.p, N + 1, nullptr);
  count_launch(c, 2);
  c->W.alloc(M);
  k_track_weight<<<ceil_div(M, T), T, 0, c->stream>>>(M, c->lm_off.p, c->e_w.p, c->W.p);
  XM_CHECK_LAUNCH();
  count_launch(c);

  phase("sort2+offsets");
  // ---- connectivity: frames ∪ observed landmarks must form one component
  {
    DBuf<int32_t>& parent = scratch_i32(c, "cc_parent");
    parent.alloc(N + M);
    k_cc_init<<<ceil_div(N + M, T), T, 0, c->stream>>>(N + M, parent.p);
    count_launch(c);
    int* d_changed = c->flags.p + 8;
    int cc_iters = 0;
    for (int it = 0; it < 100000; ++it) {
      cc_iters = it + 1;
      XM_CUDA(cudaMemsetAsync(d_changed, 0, 4, c->stream));
      k_cc_hook<<<ceil_div(Ek, T), T, 0, c->stream>>>(Ek, N, c->e_fr.p, c->e_lm.p, parent.p, d_changed);
      k_cc_jump<<<ceil_div(N + M, T), T, 0, c->stream>>>(N + M, parent.p);
      XM_CHECK_LAUNCH();
      count_launch(c, 2);
      int ch = 0;
      XM_CUDA(cudaMemcpyAsync(&ch, d_changed, 4, cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      if (!ch) break;
    }
    if (verbose) fprintf(stderr, "[xm build] connectivity iterations: %d\n", cc_iters);
    int* d_cnt = c->flags.p + 12;
    XM_CUDA(cudaMemsetAsync(d_cnt, 0, 8, c->stream));
    k_cc_count<<<ceil_div(N + M, T), T, 0, c->stream>>>(N, M, parent.p, c->lm_off.p, fcnt.p, d_cnt);
    XM_CHECK_LAUNCH();
    count_launch(c);
    int h_cc[2] = {0, 0};
    XM_CUDA(cudaMemcpyAsync(h_cc, d_cnt, 8, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (h_cc[1] > 0) throw Error(XM_EDISCONNECTED, "a frame has no observation");
    if (h_cc[0] != 1) throw Error(XM_EDISCONNECTED, "graph numerically disconnected");
  }

  phase("connectivity");
  // ---- H3: S pattern (the matrix-free mode never forms S: built on demand by
  // xm_get_S_pattern)
  // NEXT-1 (implicit.cu): Q, S, C̄ and G are never formed — only K̄, its factor
  // and inverse.  implicit_q < 0 (the default): the mode with the smaller
  // modelled time per product (the model of bench.py --mode auto)
  const bool implicit = c->opt.implicit_q > 0 || (c->opt.implicit_q < 0 && prefer_implicit(N, E, c->world));
  if (!implicit) build_s_pattern(c, N);
  else c->pattern_valid = false;

  phase("pattern");
  // ---- H4: dense S (own rows, in the Q buffer), C̄ (in the G buffer), K̄ (in L)
  const int n = 3 * N;
  c->N = N;
  c->M = M;
  c->n = n;
  c->ldq = round_up(std::max(n, 1), 32);
  c->ldk = round_up(std::max(N - 1, 1), 32);
  set_shard(c, N);
  c->implicit_active = implicit;
  if (!implicit) {
    c->Q.alloc((size_t)std::max(c->nrows, 1) * c->ldq);
    XM_CUDA(cudaMemsetAsync(c->Q.p, 0, (size_t)std::max(c->nrows, 1) * c->ldq * 8, c->stream));
  } else {
    c->Q.alloc(1);
  }
  if (N > 1) {
    c->G.alloc(implicit ? 1 : (size_t)(N - 1) * c->ldq);
    c->L.alloc((size_t)(N - 1) * c->ldk);
    if (!implicit) XM_CUDA(cudaMemsetAsync(c->G.p, 0, (size_t)(N - 1) * c->ldq * 8, c->stream));
    XM_CUDA(cudaMemsetAsync(c->L.p, 0, (size_t)(N - 1) * c->ldk * 8, c->stream));
  } else {
    c->G.alloc(1);
    c->L.alloc(1);
  }
  phase("zero S,C,K");
  if (std::getenv("XM_SCATTER_V1")) {  // round-1 kernel (A/B)
    k_clique_scatter<<<N, 128, 0, c->stream>>>(N, c->f0, c->f1, c->fr_off.p, c->fr_edge.p,
                                               c->lm_off.p, c->e_fr.p, c->e_pts.p, c->e_w.p, c->W.p,
                                               c->e_lm.p, c->Q.p, c->ldq, c->row0, c->G.p, c->L.p,
                                               c->ldk);
    XM_CHECK_LAUNCH();
    count_launch(c);
  } else {
    c->scal.alloc(64);
    double* d_T = c->scal.p + 60;
    DBuf<double>& tb = scratch_f64(c, "term_bound");
    tb.alloc(kDotBlocks);
    k_term_bound<<<kDotBlocks, 256, 0, c->stream>>>(Ek, c->e_pts.p, c->e_w.p, tb.p);
    XM_CHECK_LAUNCH();
    reduce_partials(c, tb.p, kDotBlocks, 1, d_T, 1u);  // min of −T_b
    double T = 0.0;
    XM_CUDA(cudaMemcpyAsync(&T, d_T, 8, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    T = -T;
    if (!(T > 0.0) || !std::isfinite(T)) throw Error(XM_EINVAL, "non-finite measurement scale");
    const int ex = 70 - (int)std::ceil(std::log2(T));
    const double scale = std::ldexp(1.0, ex), inv_scale = std::ldexp(1.0, -ex);
    DBuf<int32_t>& cursor = scratch_i32(c, "scatter_cursor");
    cursor.alloc(Ek);
#define XM_SCATTER_LAUNCH(WC_, NT_)                                                             \
  do {                                                                                           \
    constexpr size_t sm_ = scatter_smem<WC_, NT_>();                                             \
    ensure_smem_attr((const void*)k_clique_scatter_fx<WC_, NT_>, sm_);                           \
    k_clique_scatter_fx<WC_, NT_><<<N, NT_, sm_, c->stream>>>(                                   \
        N, c->f0, c->f1, c->world == 1 ? 1 : 0, c->fr_off.p, c->fr_edge.p, c->lm_off.p, c->e_fr.p, \
        c->e_pts.p, c->e_w.p, c->W.p, c->e_lm.p, c->Q.p, c->ldq, c->row0, c->G.p, c->L.p, c->ldk,  \
        cursor.p, scale, inv_scale, implicit ? 1 : 0);                                           \
  } while (0)
    const char* cfg = std::getenv("XM_SCATTER_CFG");
    // 768 frames × 1024 threads (213 KB, 1 CTA / SM) measured best at E and D
    // (E: 55.9 vs 60.9 ms for 384 × 512 with 2 CTAs / SM, 67 ms for 256 × 256)
    if (cfg && std::string(cfg) == "384") XM_SCATTER_LAUNCH(384, 512);
    else if (cfg && std::string(cfg) == "256") XM_SCATTER_LAUNCH(256, 256);
    else XM_SCATTER_LAUNCH(768, 1024);
#undef XM_SCATTER_LAUNCH
    XM_CHECK_LAUNCH();
    count_launch(c, 2);
  }

  phase("scatter");
  if (implicit) {
    if (N > 1) {
      DBuf<double>& U = scratch_f64(c, "chol_U");
      U.alloc((size_t)(N - 1) * c->ldk);
      dense_cholesky(c, c->L.p, N - 1, c->ldk, 1e-12, true, U.p, c->ldk);
    }
    phase("cholesky");
    implicit_prepare(c);  // frame-sorted measurements, K̄⁻¹
    phase("K^-1");
    c->have_recovery = true;
    c->normQ = implicit_normF(c);
    phase("normQ (16 probes)");
    c->stats.E = c->E;
    c->stats.q_bytes = 0;
    return;
  }
  // ---- H5: K̄ = LLᵀ, G = L⁻¹C̄, Q = S − GᵀG
  if (N > 1) {
    // pivot test relative to max diag(K̄); a disconnected graph gives a ~0 pivot
    DBuf<double>& U = scratch_f64(c, "chol_U");
    U.alloc((size_t)(N - 1) * c->ldk);
    dense_cholesky(c, c->L.p, N - 1, c->ldk, 1e-12, true, U.p, c->ldk);
    phase("cholesky");
    if (c->world == 1) {
      dense_trsm_lower_left(c, c->L.p, N - 1, c->ldk, U.p, c->ldk, c->G.p, n, c->ldq);
    } else {
      // column-sharded TRSM: G = L⁻¹C̄ splits by columns, so rank p solves
      // columns [p·w, (p+1)·w) (w a multiple of 32) and ONE all-gather of the
      // packed slices gives every rank all of G (its band rows need G up to
      // the band end; the last band needs all of it) — 3N³/P flop per rank
      // instead of 3N³, plus 8(N−1)n bytes over NVLink
      const int P = c->world, m = N - 1;
      const int w = round_up(ceil_div(n, P), 32);
      const int c0 = std::min(n, c->rank * w), c1 = std::min(n, c0 + w);
      if (c1 > c0)
        dense_trsm_lower_left(c, c->L.p, m, c->ldk, U.p, c->ldk, c->G.p + c0, c1 - c0, c->ldq);
      DBuf<double>& sl = scratch_f64(c, "trsm_slice");
      DBuf<double>& all = scratch_f64(c, "trsm_gather");
      sl.alloc((size_t)m * w);
      all.alloc((size_t)P * m * w);
      k_pack_block<<<ceil_div((int64_t)m * w, 256), 256, 0, c->stream>>>(m, w, c1 - c0, c->G.p + c0, c->ldq,
                                                                          sl.p);
      XM_CHECK_LAUNCH();
      nccl_allgather_f64(c, sl.p, all.p, (size_t)m * w);
      for (int q = 0; q < P; ++q) {
        const int q0 = std::min(n, q * w), q1 = std::min(n, q0 + w);
        if (q == c->rank || q1 <= q0) continue;
        XM_CUDA(cudaMemcpy2DAsync(c->G.p + q0, c->ldq * sizeof(double), all.p + (size_t)q * m * w,
                                  (size_t)w * sizeof(double), (size_t)(q1 - q0) * sizeof(double), m,
                                  cudaMemcpyDeviceToDevice, c->stream));
      }
      count_launch(c);
      all.release();  // 8(N−1)n bytes: not kept past the build
    }
    phase("trsm");
    const double* Gown = c->G.p + c->row0;  // columns of this rank's rows
    // Q = S − GᵀG: Q[i][j] −= Σ_k G[k][i] G[k][j]
    if (c->world == 1) {  // lower triangle + mirror: Q exactly symmetric, full storage
      dgemm_tn(c, true, n, n, N - 1, -1.0, Gown, c->ldq, c->G.p, c->ldq, 1.0, c->Q.p, c->ldq);
      mirror_lower(c, c->Q.p, n, c->ldq);
    } else if (c->nrows > 0) {  // the band's lower trapezoid: columns < row0, then its diagonal square
      dgemm_tn(c, false, c->nrows, c->row0, N - 1, -1.0, Gown, c->ldq, c->G.p, c->ldq, 1.0, c->Q.p,
               c->ldq);
      dgemm_tn(c, true, c->nrows, c->nrows, N - 1, -1.0, Gown, c->ldq, Gown, c->ldq, 1.0,
               c->Q.p + c->row0, c->ldq);
    }
  } else if (c->world == 1) {
    mirror_lower(c, c->Q.p, n, c->ldq);
  }
  phase("syrk+mirror");
  c->have_recovery = true;
  // ‖Q‖_F (all-reduced over ranks)
  {
    DBuf<double>& part = scratch_f64(c, "normq_part");
    part.alloc(kDotBlocks);
    k_sumsq_rows<<<kDotBlocks, 256, 0, c->stream>>>(c->Q.p, c->nrows, n, c->ldq, part.p,
                                                    c->world > 1 ? c->row0 : -1);
    XM_CHECK_LAUNCH();
    c->scal.alloc(64);
    reduce_partials(c, part.p, kDotBlocks, 1, c->scal.p);
    count_launch(c);
    if (c->world > 1) nccl_allreduce_sum(c, c->scal.p, 1);
    double s2 = 0.0;
    XM_CUDA(cudaMemcpyAsync(&s2, c->scal.p, 8, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    c->normQ = std::sqrt(s2);
  }
  phase("normQ");
  c->stats.E = c->E;
  c->stats.q_bytes = (int64_t)c->nrows * n * 8;
}

}  // namespace xm
