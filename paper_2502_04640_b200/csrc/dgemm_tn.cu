// dgemm_tn.cu — the dense fp64 contraction of the Q assembly (H5) on the
// fp64 tensor cores (DMMA, `mma.sync.m8n8k4.f64`), hand-written for sm_100a.
//
// Every O(N³) update of H5 has the same "TN" shape once the Cholesky factor is
// also kept transposed (U = Lᵀ, written panel by panel by the factorisation):
//
//     C[m][n] = β·C[m][n] + α · Σ_k A[k·lda + m] · B[k·ldb + n]
//
//   * Cholesky trailing update  K̄₂₂ −= L₂₁L₂₁ᵀ   : A = B = U panel (k = panel row)
//   * TRSM trailing update      C̄₂  −= L₂₁ G₁     : A = U panel, B = G block row
//   * Q = S − GᵀG (App. A)                : A = G (own columns), B = G, K = N−1
//
// so both operands are read as "k rows, contiguous m / n" and staged into
// shared memory unchanged.  Design (H5 is the one fp64-ALU-bound
// step of the path):
//   * CTA tile 128 × 128, k-block 16, 4-stage cp.async ring (16-B chunks,
//     L2-only .cg; rows / columns past the matrix are zero-filled by the copy's
//     src-size), 8 warps as 2 (m) × 4 (n), warp tile 64 × 32 = 8 × 4 DMMA
//     fragments (64 fp64 accumulators per thread).
//   * Fragment permutation: a DMMA A-fragment is A[row g][k tig]; the row of
//     m-fragment s held by lane (g, tig) is mapped to m = 16⌊s/2⌋ + 2g + (s&1),
//     so fragments s, s+1 of one k come from ONE 16-B shared load (k-major
//     tile, row pitch 132 doubles ⇒ every 8-lane phase of an LDS.128 hits 8
//     distinct 16-B bank groups).  Same for B.  The C fragment then holds 4
//     consecutive columns per (row, fragment pair): 32-B epilogue stores.
//   * TRI = 1: only tiles with tile_n ≤ tile_m (the lower triangle of a
//     symmetric result) are launched — a triangular tile enumeration, no idle
//     CTAs.
// Summation order over k is fixed (k-blocks ascending, 4 per DMMA), so the
// result is deterministic.
#include "xm_internal.cuh"

namespace xm {

namespace {

// Tile configurations: warp tile (8·FM) × 32 (FM m-fragments × 4 n-fragments),
// WMW × WNW warps.  Big: 128 × 128, 8 warps, 1 CTA / SM (the long-K SYRK of
// Q and the K = 256 TRSM updates).  Small: 64 × 64, 4 warps, 3 CTAs / SM —
// the short-K (64) Cholesky trailing updates, whose prologue / epilogue are
// then overlapped by the other resident CTAs.
template <int FM_, int WMW_, int WNW_, int BK_ = 16, int STAGES_ = 4>
struct TileCfg {
  static constexpr int FM = FM_, WMW = WMW_, WNW = WNW_;
  static constexpr int BM = WMW * 8 * FM, BN = WNW * 32, BK = BK_, STAGES = STAGES_;
  static constexpr int PITCH_A = BM + 4, PITCH_B = BN + 4;   // ≡ 4 (mod 16) doubles
  static constexpr int THREADS = 32 * WMW * WNW;
  static constexpr size_t STAGE = (size_t)BK * (PITCH_A + PITCH_B);
  static constexpr size_t SMEM = STAGE * STAGES * sizeof(double);
};
using BigTile = TileCfg<8, 2, 4>;
using BigTile32 = TileCfg<8, 2, 4, 32, 3>;   // k-block 32, 3 stages, 8 warps (A/B: XM_GEMM_TILE=w8)
using MidTile = TileCfg<8, 1, 4, 16, 4>;     // 64 × 128, 2 CTAs / SM (A/B: XM_GEMM_TILE=mid)
using W16Tile = TileCfg<4, 4, 4, 32, 3>;     // 128 × 128, 16 warps of 32 × 32: the default for
                                             // K > 64 (E: SYRK 297 vs 301 ms, TRSM 125 vs 134 ms
                                             // for 8 warps of 64 × 32, XM_GEMM_TILE=w8)
using SmallTile = TileCfg<4, 2, 2>;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Stage one k-block of a (K × ld) operand: rows k0..k0+BK−1, columns c0..c0+W−1
// into a [BK][PITCH] shared tile (zero-filled past K / C).
template <int W, int PITCH, int BK, int THREADS, bool VEC16>
__device__ __forceinline__ void load_operand(uint32_t sdst, const double* __restrict__ X, int64_t ldx,
                                             int k0, int K, int c0, int C, int tid) {
  if (VEC16) {
    constexpr int CPR = W / 2;  // 16-B chunks per row
#pragma unroll
    for (int q = 0; q < (BK * CPR) / THREADS; ++q) {
      const int ch = tid + q * THREADS;
      const int kk = ch / CPR, cc = (ch % CPR) * 2;
      const int gk = k0 + kk, gc = c0 + cc;
      int bytes = 0;
      const double* src = X;
      if (gk < K && gc < C) {
        bytes = min(2, C - gc) * 8;
        src = X + (int64_t)gk * ldx + gc;
      }
      cp_async16(sdst + (uint32_t)(kk * PITCH + cc) * 8u, src, bytes);
    }
  } else {
#pragma unroll
    for (int q = 0; q < (BK * W) / THREADS; ++q) {
      const int ch = tid + q * THREADS;
      const int kk = ch / W, cc = ch % W;
      const int gk = k0 + kk, gc = c0 + cc;
      const bool ok = gk < K && gc < C;
      cp_async8(sdst + (uint32_t)(kk * PITCH + cc) * 8u, ok ? X + (int64_t)gk * ldx + gc : X,
                ok ? 8 : 0);
    }
  }
}

template <class T, int TRI, bool VEC16>
__global__ void __launch_bounds__(T::THREADS)
    k_dgemm_tn(int M, int N, int K, double alpha, const double* __restrict__ A, int64_t lda,
               const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C,
               int64_t ldc, int tiles_n, int vec_out) {
  constexpr int FM = T::FM, BK = T::BK, ST = T::STAGES, PA = T::PITCH_A, PB = T::PITCH_B;
  extern __shared__ __align__(16) double smem[];
  int tm, tn;
  if (TRI) {  // triangular enumeration t = tm(tm+1)/2 + tn, tn ≤ tm
    const int64_t t = blockIdx.x;
    int a = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((int64_t)(a + 1) * (a + 2) / 2 <= t) ++a;
    while ((int64_t)a * (a + 1) / 2 > t) --a;
    tm = a;
    tn = (int)(t - (int64_t)a * (a + 1) / 2);
  } else {
    tm = blockIdx.x / tiles_n;
    tn = blockIdx.x % tiles_n;
  }
  const int m0 = tm * T::BM, n0 = tn * T::BN;
  // TRI == 2: A = B lower triangular in (k, m) (A[k][m] = 0 for k < m, e.g.
  // X = L⁻¹ read transposed): the output rows m ≥ m0 only see k ≥ m0
  const int kbeg = (TRI == 2) ? m0 / BK : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp % T::WMW, wn = warp / T::WMW;

  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  auto sA = [&](int st) { return sbase + (uint32_t)(st * T::STAGE) * 8u; };
  auto sB = [&](int st) { return sbase + (uint32_t)(st * T::STAGE + BK * PA) * 8u; };
  auto load = [&](int st, int kb) {
    load_operand<T::BM, PA, BK, T::THREADS, VEC16>(sA(st), A, lda, kb * BK, K, m0, M, tid);
    load_operand<T::BN, PB, BK, T::THREADS, VEC16>(sB(st), B, ldb, kb * BK, K, n0, N, tid);
  };

  double acc[FM][4][2];
#pragma unroll
  for (int s = 0; s < FM; ++s)
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

  const int nk = (K + BK - 1) / BK - kbeg;
#pragma unroll
  for (int st = 0; st < ST - 1; ++st) {
    if (st < nk) load(st, kbeg + st);
    cp_commit();
  }
  // per-lane shared offsets (doubles) of its fragment pairs
  const int a_off = tig * PA + wm * 8 * FM + 2 * g;
  const int b_off = tig * PB + wn * 32 + 2 * g;
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<ST - 2>();
    __syncthreads();
    {  // refill the slot consumed in iteration kt−1
      const int nx = kt + ST - 1;
      if (nx < nk) load(nx % ST, kbeg + nx);
      cp_commit();
    }
    const double* As = smem + (kt % ST) * T::STAGE;
    const double* Bs = As + BK * PA;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[FM], b[4];
#pragma unroll
      for (int q = 0; q < FM / 2; ++q) {
        const double2 v = *reinterpret_cast<const double2*>(As + ks * 4 * PA + a_off + 16 * q);
        a[2 * q] = v.x;
        a[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double2 v = *reinterpret_cast<const double2*>(Bs + ks * 4 * PB + b_off + 16 * q);
        b[2 * q] = v.x;
        b[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int s = 0; s < FM; ++s)
#pragma unroll
        for (int t = 0; t < 4; ++t) dmma(acc[s][t][0], acc[s][t][1], a[s], b[t]);
    }
  }
  cp_wait<0>();

  // epilogue: fragment s row g → m = m0 + 8·FM·wm + 16⌊s/2⌋ + 2g + (s&1);
  // fragment t, element e → n = n0 + 32wn + 16⌊t/2⌋ + 4tig + 2e + (t&1)
#pragma unroll
  for (int s = 0; s < FM; ++s) {
    const int m = m0 + wm * 8 * FM + 16 * (s >> 1) + 2 * g + (s & 1);
    if (m >= M) continue;
    double* crow = C + (int64_t)m * ldc;
#pragma unroll
    for (int tp = 0; tp < 2; ++tp) {
      const int nb = n0 + wn * 32 + 16 * tp + 4 * tig;
      double v[4] = {acc[s][2 * tp][0], acc[s][2 * tp + 1][0], acc[s][2 * tp][1],
                     acc[s][2 * tp + 1][1]};
      if (vec_out && nb + 3 < N) {
        double4* p = reinterpret_cast<double4*>(crow + nb);
        double4 o = make_double4(0.0, 0.0, 0.0, 0.0);
        if (beta != 0.0) o = *p;
        o.x = fma(alpha, v[0], beta * o.x);
        o.y = fma(alpha, v[1], beta * o.y);
        o.z = fma(alpha, v[2], beta * o.z);
        o.w = fma(alpha, v[3], beta * o.w);
        *p = o;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int n = nb + e;
          if (n < N) {
            const double old = beta != 0.0 ? crow[n] : 0.0;
            crow[n] = fma(alpha, v[e], beta * old);
          }
        }
      }
    }
  }
}

template <class T, int TRI, bool V>
void launch_tn(xm_ctx* c, int M, int N, int K, double alpha, const double* A, int64_t lda,
               const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  ensure_smem_attr((const void*)k_dgemm_tn<T, TRI, V>, T::SMEM);
  const int tm = ceil_div(M, T::BM), tn = ceil_div(N, T::BN);
  const int64_t tiles = TRI ? (int64_t)tm * (tm + 1) / 2 : (int64_t)tm * tn;  // TRI 1, 2: lower tiles
  if (tiles <= 0) return;
  if (tiles > INT32_MAX) throw Error(XM_EINVAL, "dgemm_tn: too many tiles");
  const int vec_out = ((reinterpret_cast<uintptr_t>(C) & 31) == 0 && (ldc & 3) == 0) ? 1 : 0;
  k_dgemm_tn<T, TRI, V><<<(unsigned)tiles, T::THREADS, T::SMEM, c->stream>>>(
      M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, tn, vec_out);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

template <class T>
void dispatch(xm_ctx* c, bool lower, bool v16, int M, int N, int K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  if (lower) {
    if (v16) launch_tn<T, 1, true>(c, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else launch_tn<T, 1, false>(c, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  } else {
    if (v16) launch_tn<T, 0, true>(c, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else launch_tn<T, 0, false>(c, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  }
}

}  // namespace

// C (lower tiles) = α XᵀX + β C for X lower triangular (X[k][m] = 0 for k < m):
// the k-loop of output row block m0 starts at m0 — m³/3 instead of m³ flops
// (NEXT-1: K̄⁻¹ = L⁻ᵀL⁻¹, implicit.cu)
void dsyrk_tn_lowtri(xm_ctx* c, int M, double alpha, const double* X, int64_t ldx, double beta, double* C,
                     int64_t ldc) {
  if (M <= 0) return;
  const bool v16 = (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (ldx % 2) == 0;
  if (v16) launch_tn<W16Tile, 2, true>(c, M, M, M, alpha, X, ldx, X, ldx, beta, C, ldc);
  else launch_tn<W16Tile, 2, false>(c, M, M, M, alpha, X, ldx, X, ldx, beta, C, ldc);
}

void dgemm_tn(xm_ctx* c, bool lower, int M, int N, int K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    if (beta == 1.0) return;
    K = 0;
  }
  if (lower && M != N) throw Error(XM_EINVAL, "dgemm_tn: lower needs M == N");
  const bool v16 = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                   (lda % 2) == 0 && (ldb % 2) == 0;
  // short K (the Cholesky's rank-64 updates): small tiles, several CTAs per SM
  if (K <= 64) dispatch<SmallTile>(c, lower, v16, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (c->gemm_tile == 1) dispatch<BigTile>(c, lower, v16, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (c->gemm_tile == 2 && !lower) dispatch<MidTile>(c, lower, v16, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (c->gemm_tile == 3) dispatch<BigTile32>(c, lower, v16, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else dispatch<W16Tile>(c, lower, v16, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

}  // namespace xm
