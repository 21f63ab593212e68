// spmm_sym.cu — H6 with symmetric Q: out = Q·V streaming only the lower
// triangle (Q = Qᵀ by construction, Prop. 1) — half the HBM bytes of the
// full-row kernel (spmm.cu).
//
//   out_i = Σ_{j ≤ i} Q_ij V_j  +  Σ_{j > i} Q_ji V_j
//         = row part (lower triangle) + column part (strictly lower triangle)
//
// Geometry (column-strip order).  The lower triangle is cut into column
// panels J of BC = 256 columns; panel J is the run of TR = 32-row tiles that
// start at its diagonal block (row tiles 8J … ⌈n/32⌉−1).  Tiles are numbered
// panel-major and the W tiles are split stream-K style into G = 148 equal
// contiguous ranges (one persistent CTA per SM).  A CTA's range is a short
// sequence of *segments* (runs of tiles of one panel; 1–3 per CTA at the
// bench sizes), so:
//   * V_J for the lane's 8 columns and the column partials stay in registers
//     for the whole segment — one column partial per segment (negligible
//     traffic), not one per tile;
//   * the row part of a tile is a finished 32 × r partial of (rows, panel J),
//     written once (rowpart[tile]): R/256 extra bytes per Q byte.
//
// Per tile (warp w ↔ rows 4w … 4w+3; lane ℓ ↔ the 8 columns {2ℓ+64m, 2ℓ+64m+1},
// m = 0..3 — conflict-free LDS.128):
//   row part   r_i += Σ_j Q_ij V_j over the lane's columns for RP rows at a
//              time, then ONE butterfly reduce-scatter over the warp for the
//              RP rows together (xor 16 / 8 halve the row set, the remaining
//              levels sum): 6r shuffles per 4 rows instead of 5r per row;
//   column part c_j += Q_ij V_i (j < i), accumulated in registers over the
//              segment (V_i broadcast from shared memory).
// Thread 0 streams each tile with ONE 2-D tensor TMA copy (box 256 × 32, L2
// evict-first; rows / columns past n zero-filled) plus the tile's 32 × r
// slice of V (1-D bulk copy) into a 3-stage ring (3 × 65 KB).
//
// After a software grid barrier the same CTAs sum, in a fixed order, the row
// parts of the tiles (K, J ≤ ⌊row/256⌋) and the column parts of the segments
// of panel ⌊row/256⌋ (consecutive segment numbers), and apply the per-camera
// epilogue (same modes as spmm.cu).  Deterministic; algorithmic bytes per
// product: 8·n(n+1)/2 + 16·n·r.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "frame_ops.cuh"

#include <map>
#include <type_traits>

namespace xm {

namespace {
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int BC = 256;                  // panel width (columns)
constexpr int TR = 32;                   // rows per tile (4 per consumer warp)
constexpr int kRowsPerWarp = TR / kWarps;
constexpr int kDiagTiles = BC / TR;      // tiles of a panel's diagonal block
constexpr int kTileBytes = TR * BC * 8;  // 64 KB
constexpr int kStages = 3;
constexpr int kVsliceDoubles = TR * 6;   // V_I slice (r ≤ 5), padded; stage stride stays 128-B aligned
constexpr int kStageDoubles = TR * BC + kVsliceDoubles;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(cnt));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;\n" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(b)), "l"(pol)
      : "memory");
}
// 2-D tensor copy of one TR × BC tile of Q (OOB rows / columns zero-filled)
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* b,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(su32(b)), "l"(pol)
      : "memory");
}
// tile t → panel J using pbase[J] = Σ_{J'<J} (TRt − 8J')
__device__ __forceinline__ int tile_panel(int64_t t, const int* __restrict__ pbase, int TCb) {
  int lo = 0, hi = TCb - 1;
  while (lo < hi) {  // largest J with pbase[J] ≤ t
    int mid = (lo + hi + 1) >> 1;
    if (pbase[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// First row-part slot of row tile K: Σ_{K'<K} (⌊K'/8⌋ + 1) (panels 0..⌊K'/8⌋
// intersect row tile K'), so the row parts of one row tile are contiguous.
__device__ __forceinline__ int64_t rtile_base(int K) {
  const int64_t a = K >> 3, b = K & 7;
  return (int64_t)K + 4 * a * (a - 1) + a * b;
}

// Butterfly reduce-scatter of RP rows × R partial sums over the 32 lanes:
// on return lane ℓ holds the full sums of row ((ℓ >> (5 − log2 RP)) & (RP−1))
// in a[0][·].  Fixed order ⇒ deterministic.
template <int RP, int R>
__device__ __forceinline__ void warp_rows_reduce(double (&a)[RP][R], int lane) {
  if constexpr (RP == 4) {
    const bool h16 = (lane & 16) != 0;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) {
        const double snd = h16 ? a[k][cc] : a[k + 2][cc];
        const double kp = h16 ? a[k + 2][cc] : a[k][cc];
        a[k][cc] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
      }
  }
  if constexpr (RP >= 2) {
    constexpr int o = (RP == 4) ? 8 : 16;
    const bool hb = (lane & o) != 0;
#pragma unroll
    for (int cc = 0; cc < R; ++cc) {
      const double snd = hb ? a[0][cc] : a[1][cc];
      const double kp = hb ? a[1][cc] : a[0][cc];
      a[0][cc] = kp + __shfl_xor_sync(0xffffffffu, snd, o);
    }
  }
  constexpr int top = (RP == 4) ? 4 : (RP == 2 ? 8 : 16);
#pragma unroll
  for (int o = top; o > 0; o >>= 1)
#pragma unroll
    for (int cc = 0; cc < R; ++cc) a[0][cc] += __shfl_xor_sync(0xffffffffu, a[0][cc], o);
}
}  // namespace

// Static work plan for one (n, G): panel bases, per-CTA segment bases and the
// first segment of every panel (segments are numbered in tile order, so the
// segments of one panel are consecutive — fixed summation order for the finish).
struct SymPlan {
  int n = 0, G = 0, TRt = 0, TCb = 0, S = 0;
  int rt_a = 0, rt_b = 0, row0 = 0;  // this rank's band of row tiles (one GPU: all of them)
  int64_t W = 0, W_full = 0;         // tiles of the band / of the whole lower triangle
  const void* qptr = nullptr;  // Q the tensor map was encoded for
  int64_t ldq = 0;
  CUtensorMap tmq;
  DBuf<int> pbase;    // TCb + 1
  DBuf<int> segbase;  // G + 1
  DBuf<int> colptr;   // TCb + 1: segments [colptr[J], colptr[J+1]) belong to panel J
};

// The symmetric matrix a plan streams: Q (this rank's band of rows) or, in
// the matrix-free mode, K̄⁻¹ (implicit.cu) — any n × n symmetric matrix whose
// rows [row0, row0 + nrows) are stored with pitch ld (lower triangle read).
struct SymSrc {
  const double* ptr;
  int n;
  int64_t ld;
  int row0, nrows;
};

static SymPlan& sym_plan_for(xm_ctx* c, void*& slot, const SymSrc& src) {
  if (!slot) slot = new SymPlan();
  SymPlan& p = *static_cast<SymPlan*>(slot);
  int sms = 148;
  XM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const int n = src.n, G = std::min(148, sms);
  // band of row tiles: [row0, row0 + nrows) is frame- and tile-aligned (32 frames) on world > 1
  const int rt_a = src.row0 / TR;
  const int rt_b = (src.row0 + src.nrows >= n) ? ceil_div(n, TR) : (src.row0 + src.nrows) / TR;
  const bool same_band = p.rt_a == rt_a && p.rt_b == rt_b && p.row0 == src.row0;
  if (p.n == n && p.G == G && p.pbase.p && p.qptr == src.ptr && p.ldq == src.ld && same_band) return p;
  // Q tensor map: dims {n columns, n rows}, row pitch ldq·8 B, box BC × TR,
  // OOB → zero fill (rows / columns ≥ n read as 0)
  {
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&f),
                                  cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        f = nullptr;
      return f;
    }();
    if (!encode) throw Error(XM_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)std::max(src.nrows, 1)};  // local rows
    cuuint64_t strides[1] = {(cuuint64_t)src.ld * 8};
    cuuint32_t box[2] = {(cuuint32_t)BC, (cuuint32_t)TR};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&p.tmq, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(src.ptr), dims,
                        strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(XM_ECUDA, "cuTensorMapEncodeTiled failed");
    p.qptr = src.ptr;
    p.ldq = src.ld;
  }
  if (p.n == n && p.G == G && p.pbase.p && same_band) return p;
  p.n = n;
  p.G = G;
  p.TRt = ceil_div(n, TR);
  p.TCb = ceil_div(n, BC);
  p.rt_a = rt_a;
  p.rt_b = rt_b;
  p.row0 = src.row0;
  // panel J: row tiles max(8J, rt_a) … rt_b − 1 of the band (none once 8J ≥ rt_b)
  std::vector<int> pb(p.TCb + 1, 0);
  for (int J = 0; J < p.TCb; ++J)
    pb[J + 1] = pb[J] + std::max(0, rt_b - std::max(kDiagTiles * J, rt_a));
  p.W = pb[p.TCb];
  p.W_full = 0;
  for (int J = 0; J < p.TCb; ++J) p.W_full += p.TRt - kDiagTiles * J;
  std::vector<int> segbase(G + 1, 0), segpanel;
  for (int cta = 0; cta < G; ++cta) {
    const int64_t t0 = (int64_t)cta * p.W / G, t1 = (int64_t)(cta + 1) * p.W / G;
    segbase[cta] = (int)segpanel.size();
    int J = 0;
    while (J + 1 < p.TCb && pb[J + 1] <= t0) ++J;
    for (int64_t t = t0; t < t1;) {
      while (pb[J + 1] <= t) ++J;
      segpanel.push_back(J);
      t = std::min<int64_t>(t1, pb[J + 1]);
    }
  }
  segbase[G] = (int)segpanel.size();
  p.S = (int)segpanel.size();
  std::vector<int> colptr(p.TCb + 1, 0);
  for (int s = 0, J = 0; J <= p.TCb; ++J) {  // segpanel is non-decreasing
    while (s < p.S && segpanel[s] < J) ++s;
    colptr[J] = s;
  }
  p.pbase.alloc(pb.size());
  p.segbase.alloc(segbase.size());
  p.colptr.alloc(colptr.size());
  XM_CUDA(cudaMemcpy(p.pbase.p, pb.data(), pb.size() * 4, cudaMemcpyHostToDevice));
  XM_CUDA(cudaMemcpy(p.segbase.p, segbase.data(), segbase.size() * 4, cudaMemcpyHostToDevice));
  XM_CUDA(cudaMemcpy(p.colptr.p, colptr.data(), colptr.size() * 4, cudaMemcpyHostToDevice));
  return p;
}

static SymPlan& sym_plan(xm_ctx* c) {
  return sym_plan_for(c, c->sym_plan, SymSrc{c->Q.p, (int)c->n, c->ldq, c->row0, c->nrows});
}

template <int R>
struct SymCfg {
#ifndef XM_SYM_RP4_MAXR
#define XM_SYM_RP4_MAXR 4
#endif
  static constexpr int kRP = (R <= XM_SYM_RP4_MAXR) ? 4 : 2;  // rows reduced together (register budget)
  static constexpr size_t kSmem =
      (size_t)kStages * kStageDoubles * 8 + (size_t)BC * R * 8 + 64 * 8;
};

template <int R, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_spmm_sym(
    const __grid_constant__ CUtensorMap tmq, int N, int n, int rt_a, int rt_b, int row0, int TCb,
    int64_t W,
    const int* __restrict__ pbase, const int* __restrict__ segbase, const int* __restrict__ colptr,
    const double* __restrict__ V, double* __restrict__ rowpart, double* __restrict__ colpart,
    GridBar* __restrict__ gbar, SpmmEpiArgs ep) {
  using Cfg = SymCfg<R>;
  constexpr int RP = Cfg::kRP;
  if (ep.stop && *ep.stop) return;
  if (ep.exec && blockIdx.x == 0 && threadIdx.x == 0) *ep.exec = 1;
  extern __shared__ __align__(128) unsigned char sm[];
  double* stages = reinterpret_cast<double*>(sm);
  double* colred = stages + (size_t)kStages * kStageDoubles;  // [BC][R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(colred + BC * R);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;

  const int G = gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * W / G;
  const int64_t t1 = (int64_t)(blockIdx.x + 1) * W / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ------------------------------------------------------------ producer
  // Thread 0 (of consumer warp 0) issues the loads: the first kStages tiles
  // here, then tile it + kStages into slot it % kStages once all 8 warps have
  // released tile it.  No separate producer warp: 8 warps = 2 per SM
  // sub-partition, so each thread may use up to 255 registers (9 warps would
  // put 3 warps on one sub-partition and cap the kernel at 168).
  int pJ = 0, ppend = 0;
  int64_t pt_next = t0;
  uint64_t pq = 0, pv = 0;
  auto issue = [&](int it_load) {
    const int64_t t = pt_next++;
    if (t >= ppend) {
      ++pJ;
      ppend = pbase[pJ + 1];
    }
    const int rt = max(kDiagTiles * pJ, rt_a) + (int)(t - pbase[pJ]);  // row tile (global)
    const int s = it_load % kStages;
    const int ni = min(TR, n - rt * TR);
    const unsigned bv = (unsigned)(((ni * R + 1) & ~1) * 8);
    bar_expect(&full[s], (unsigned)kTileBytes + bv);
    double* st = stages + (size_t)s * kStageDoubles;
    tma_tile(st, &tmq, pJ * BC, rt * TR - row0, &full[s], pq);  // local row of this rank's Q
    bulk_g2s(st + TR * BC, V + (int64_t)rt * TR * R, bv, &full[s], pv);
  };
  const int ntiles = (int)(t1 - t0);
  if (threadIdx.x == 0 && ntiles > 0) {
    pq = pol_first();
    pv = pol_last();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmq)) : "memory");
    pJ = tile_panel(t0, pbase, TCb) - 1;
    ppend = pbase[pJ + 1];
    for (int k = 0; k < min(kStages, ntiles); ++k) issue(k);
  }
  {
    // ------------------------------------------------------------ consumers
    double vr[8][R];      // V_J rows for the lane's 8 columns (whole segment)
    double colacc[8][R];  // column partials for the lane's 8 columns
    int seg = 0, J = -1, pend = 0;
    int it = 0;
    auto flush = [&]() {
      // fixed-order cross-warp sum of colacc (warp 0 stores, warps 1..7 add in
      // turn), then the segment's column partial is written out
#pragma unroll 1
      for (int w = 0; w < kWarps; ++w) {
        if (warp == w) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int cc = 0; cc < R; ++cc) {
                double* d = &colred[(2 * lane + 64 * m + h) * R + cc];
                *d = (w == 0) ? colacc[2 * m + h][cc] : *d + colacc[2 * m + h][cc];
              }
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kWarps) : "memory");
      }
      double* dst = colpart + ((int64_t)(segbase[blockIdx.x] + seg - 1)) * BC * R;
      for (int e = threadIdx.x; e < BC * R; e += 32 * kWarps) dst[e] = colred[e];
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kWarps) : "memory");
    };
    // RP rows (k0 … k0+RP−1 of the warp's 4) of one tile
    auto do_rows = [&](auto diag_tag, const double* st, const double* vi, int nv, int k0, int dl0,
                       double* rp) {
      constexpr bool DIAG = decltype(diag_tag)::value;
      double rs[RP][R];
#pragma unroll
      for (int k = 0; k < RP; ++k) {
        const int rl = kRowsPerWarp * warp + k0 + k;  // row within the tile
        const double* q = st + rl * BC;
        double vrow[R];
#pragma unroll
        for (int cc = 0; cc < R; ++cc) vrow[cc] = (rl < nv) ? vi[rl * R + cc] : 0.0;
        const int dl = dl0 + rl;  // diagonal column within the panel (DIAG only)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) rs[k][cc] = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int jl = 2 * lane + 64 * m;
          const double2 q2 = *reinterpret_cast<const double2*>(q + jl);
          double qa = q2.x, qb = q2.y, ca = qa, cb = qb;
          if (DIAG) {  // row part j ≤ i, column part j < i; beyond: zero
            qa = (jl <= dl) ? qa : 0.0;
            qb = (jl + 1 <= dl) ? qb : 0.0;
            ca = (jl < dl) ? q2.x : 0.0;
            cb = (jl + 1 < dl) ? q2.y : 0.0;
          }
#pragma unroll
          for (int cc = 0; cc < R; ++cc) {
            rs[k][cc] = fma(qa, vr[2 * m][cc], fma(qb, vr[2 * m + 1][cc], rs[k][cc]));
            colacc[2 * m][cc] = fma(ca, vrow[cc], colacc[2 * m][cc]);
            colacc[2 * m + 1][cc] = fma(cb, vrow[cc], colacc[2 * m + 1][cc]);
          }
        }
      }
      warp_rows_reduce<RP, R>(rs, lane);
      constexpr int sh = (RP == 4) ? 3 : (RP == 2 ? 4 : 5);
      if ((lane & ((1 << sh) - 1)) == 0) {
        const int rl = kRowsPerWarp * warp + k0 + (lane >> sh);
#pragma unroll
        for (int cc = 0; cc < R; ++cc) rp[rl * R + cc] = rs[0][cc];
      }
    };
    for (int64_t t = t0; t < t1; ++t, ++it) {
      if (t >= pend) {  // new segment (panel J): flush the previous one, load V_J
        if (J >= 0) flush();
        J = (J < 0) ? tile_panel(t0, pbase, TCb) : J + 1;
        pend = pbase[J + 1];
        const int nj = min(BC, n - J * BC);
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jl = 2 * lane + 64 * m + h;
#pragma unroll
            for (int cc = 0; cc < R; ++cc) {
              vr[2 * m + h][cc] = (jl < nj) ? V[((int64_t)J * BC + jl) * R + cc] : 0.0;
              colacc[2 * m + h][cc] = 0.0;
            }
          }
        ++seg;
      }
      const int rt = max(kDiagTiles * J, rt_a) + (int)(t - pbase[J]);  // row tile (global)
      const int pt = rt - kDiagTiles * J;  // tile index within the full panel (< 8: diagonal block)
      const int s = it % kStages;
      bar_wait(&full[s], (unsigned)((it / kStages) & 1));
      const double* st = stages + (size_t)s * kStageDoubles;
      const double* vi = st + TR * BC;
      const int nv = n - rt * TR;  // rows ≥ n: Q reads as 0 (TMA zero fill), V slice is short
      double* rp = rowpart + (rtile_base(rt) + J) * TR * R;  // [row tile][panel] order
#ifndef XM_EXP_NOCOMPUTE
      if (pt < kDiagTiles) {
#pragma unroll
        for (int k0 = 0; k0 < kRowsPerWarp; k0 += RP) do_rows(std::true_type{}, st, vi, nv, k0, pt * TR, rp);
      } else {
#pragma unroll
        for (int k0 = 0; k0 < kRowsPerWarp; k0 += RP) do_rows(std::false_type{}, st, vi, nv, k0, 0, rp);
      }
#else
      (void)rp; (void)pt;
#endif
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[s]);
      if (threadIdx.x == 0 && it + kStages < ntiles) {  // refill slot s once every warp released it
        bar_wait(&empty[s], (unsigned)((it / kStages) & 1));
        issue(it + kStages);
      }
    }
    if (J >= 0) flush();
  }

  // ------------------------------------------------------------ finish (fused)
  // All row / column partials are published; CTA c now sums, for the rows of
  // frames [c·N/G, (c+1)·N/G), the row parts of panels 0..⌊row/256⌋ (stored
  // contiguously per row tile) and the column parts of the segments of panel
  // ⌊row/256⌋, one (row, column) element per thread in a fixed order
  // (coalesced across threads), then applies the per-camera epilogue.
#ifdef XM_EXP_NOFINISH
  return;
#endif
  grid_barrier(gbar, G);
  const int fa = (int)((int64_t)blockIdx.x * N / G), fb = (int)((int64_t)(blockIdx.x + 1) * N / G);
  double* qrow = stages;  // pipeline smem is free now: [rows][R]
  for (int e = threadIdx.x; e < 3 * (fb - fa) * R; e += kThreads) {
    const int row = 3 * fa + e / R, cc = e % R;
    if (row >= n) {  // a matrix of order n < 3N (K̄⁻¹): the padding rows read as 0
      qrow[e] = 0.0;
      continue;
    }
    const int K = row / TR, l = row % TR;
    const int Jc = row / BC, m = row % BC;
    const double* p = rowpart + (rtile_base(K) * TR + l) * R + cc;
    double acc = 0.0;
    int q = (K >= rt_a && K < rt_b) ? 0 : Jc + 1;  // row parts exist for the band's rows only
#ifndef XM_SYM_FIN_INFLIGHT
#define XM_SYM_FIN_INFLIGHT 32
#endif
    constexpr int kF = XM_SYM_FIN_INFLIGHT;
    for (; q + kF <= Jc + 1; q += kF) {  // kF loads in flight, summed in order (the
      // finish is latency-bound: ≈ n/256 partials per element, one element per thread)
      double v[kF];
#pragma unroll
      for (int u = 0; u < kF; ++u) v[u] = p[(int64_t)(q + u) * TR * R];
#pragma unroll
      for (int u = 0; u < kF; ++u) acc += v[u];
    }
    if (kF > 16 && q + 16 <= Jc + 1) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = p[(int64_t)(q + u) * TR * R];
#pragma unroll
      for (int u = 0; u < 16; ++u) acc += v[u];
      q += 16;
    }
    for (; q + 4 <= Jc + 1; q += 4) {  // 4 loads in flight, summed in order
      const double a0 = p[(int64_t)q * TR * R], a1 = p[(int64_t)(q + 1) * TR * R];
      const double a2 = p[(int64_t)(q + 2) * TR * R], a3 = p[(int64_t)(q + 3) * TR * R];
      acc = (((acc + a0) + a1) + a2) + a3;
    }
    for (; q <= Jc; ++q) acc += p[(int64_t)q * TR * R];
    for (int sg = colptr[Jc]; sg < colptr[Jc + 1]; ++sg) acc += colpart[((int64_t)sg * BC + m) * R + cc];
    qrow[e] = acc;
  }
  __syncthreads();
  constexpr int NC = (MODE == EPI_GRAD) ? 3 : (MODE == EPI_DF ? 2 : 1);
  double pt[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) pt[q] = (MODE == EPI_GRAD && q == 2) ? 1.0e300 : 0.0;
  for (int lf = threadIdx.x; lf < fb - fa; lf += kThreads) {
    const int i = fa + lf;
    Blk<R> qv;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) qv.v[a][cc] = qrow[(3 * lf + a) * R + cc];
    if (MODE == EPI_STORE) {
      store_blk<R>(ep.out, i, qv);
    } else if (MODE == EPI_HVP) {
      Blk<R> y, vv, w;
      load_blk<R>(ep.Y, i, y);
      load_blk<R>(V, i, vv);
      double L[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) L[q] = ep.lam[6 * i + q];
      sub_lam<R>(qv, L, vv, 2.0, 2.0, w);
      project_blk<R>(y, i == 0, w);
      store_blk<R>(ep.out2, i, w);
      pt[0] += dotb<R>(vv, w);
    } else if (MODE == EPI_ZMUL) {
      Blk<R> vv, w;
      load_blk<R>(V, i, vv);
      double L[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) L[q] = ep.lam[6 * i + q];
      sub_lam<R>(qv, L, vv, 1.0, 1.0, w);
      store_blk<R>(ep.out, i, w);
      pt[0] += dotb<R>(vv, w);
    } else if (MODE == EPI_DF) {
      Blk<R> d, qy;
      load_blk<R>(V, i, d);
      load_blk<R>(ep.aux, i, qy);
      store_blk<R>(ep.out, i, qv);
      pt[0] += dotb<R>(qy, d);
      pt[1] += dotb<R>(d, qv);
    } else if (MODE == EPI_GRAD) {
      Blk<R> y, gr;
      load_blk<R>(V, i, y);
      store_blk<R>(ep.out, i, qv);
      double M[3][3], L[6];
      mul_abt<R>(qv, y, M);
      double alpha = frob2<R>(y) / 3.0;
      sym_lambda(M, i == 0, alpha, L);
#pragma unroll
      for (int q = 0; q < 6; ++q) ep.lam_out[6 * i + q] = L[q];
      sub_lam<R>(qv, L, y, 2.0, 2.0, gr);
      store_blk<R>(ep.out2, i, gr);
      pt[0] += dotb<R>(y, qv);
      pt[1] += frob2<R>(gr);
      if (i > 0) pt[2] = fmin(pt[2], alpha);
    }
  }
  if (MODE != EPI_STORE) block_reduce_store<NC, kThreads>(pt, ep.partials, MODE == EPI_GRAD ? 4u : 0u);
}

// ---------------------------------------------------------------- host side
// Kernel choice per (N, r), from tools/exp_sym.sh on B200.
void sym_plan_destroy(xm_ctx* c) {
  delete static_cast<SymPlan*>(c->sym_plan);
  c->sym_plan = nullptr;
}

// Every plain product (gradient, Δf, Lanczos, HVP outside the persistent tCG)
// takes the lower-triangle kernel on one GPU: measured faster than the
// full-row stream at every (N, r) (B: 40.8 vs 55.4 µs at r = 3; E: 587 vs
// 1037 µs at r = 3, 676 vs 1227 at r = 4).  The tCG loop keeps the persistent
// full-row kernel below N = 4000 (tcg_fullrow_ok), where one fused launch per
// TR step beats a three-kernel iteration around this one.
bool spmm_sym_supported(xm_ctx* c, int r) {
  if (r < 1 || r > 5) return false;
  if (c->world > 1) return true;  // the band layout stores only the lower trapezoid
  return c->opt.spmm_kernel != 1;
}

bool tcg_fullrow_ok(xm_ctx* c) { return c->opt.spmm_kernel != 2 && c->N < 4000; }

int spmm_sym_partials(xm_ctx* c) { return sym_plan(c).G; }

// part: row / column partials, sized once for the largest supported r so the
// address never changes when the staircase climbs (the tCG graphs of lower
// ranks captured it).  Nf = frames of the finish (3 rows each; rows ≥ n skipped).
template <int R, int MODE>
static void launch_sym_on(xm_ctx* c, SymPlan& p, DBuf<double>& part, int Nf, const double* V,
                          const SpmmEpiArgs& ep) {
  constexpr int kRmax = 5;
  const size_t rp = (size_t)p.W_full * TR * R;  // row parts indexed over the whole triangle
  part.alloc((size_t)p.W_full * TR * kRmax + (size_t)std::max(p.S, 1) * BC * kRmax + 64);
  double* rowpart = part.p;
  double* colpart = part.p + rp;
  if (!c->gbar.p) {
    c->gbar.alloc(4);
    XM_CUDA(cudaMemset(c->gbar.p, 0, 4 * sizeof(int)));
  }
  const size_t smem = SymCfg<R>::kSmem;
  ensure_smem_attr((const void*)k_spmm_sym<R, MODE>, smem);
  // grid barrier inside: a cooperative launch guarantees (or cleanly refuses)
  // the co-residency of the p.G CTAs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  XM_CUDA(cudaLaunchKernelEx(&cfg, k_spmm_sym<R, MODE>, p.tmq, Nf, p.n, p.rt_a, p.rt_b, p.row0, p.TCb,
                             p.W, p.pbase.p, p.segbase.p, p.colptr.p, V, rowpart, colpart,
                             reinterpret_cast<GridBar*>(c->gbar.p), ep));
  XM_CHECK_LAUNCH();
  count_launch(c, 1);
}

template <int R, int MODE>
static void launch_sym(xm_ctx* c, const double* V, const SpmmEpiArgs& ep) {
  launch_sym_on<R, MODE>(c, sym_plan(c), c->sym_part, (int)c->N, V, ep);
}

// out = A·V for a symmetric m × m matrix A (pitch lda, lower triangle read),
// V and out m × r row-major with ≥ 3·⌈m/3⌉ rows of room (r ≤ 5).  NEXT-1:
// the K̄⁻¹ product of the matrix-free Q·V (implicit.cu).
void spmm_sym_matrix(xm_ctx* c, void*& plan_slot, DBuf<double>& part, const double* A, int m,
                     int64_t lda, const double* V, int r, double* out, const int* stop, int row0,
                     int nrows) {
  // band [row0, row0 + nrows) (32-row aligned; world > 1): the partial of its
  // lower trapezoid, full length (row parts of its rows, column parts above)
  if (nrows < 0) nrows = m;
  SymPlan& p = sym_plan_for(c, plan_slot, SymSrc{A + (int64_t)row0 * lda, m, lda, row0, nrows});
  SpmmEpiArgs ep{};
  ep.out = out;
  ep.stop = stop;
  const int Nf = ceil_div(m, 3);
  switch (r) {
    case 1: launch_sym_on<1, EPI_STORE>(c, p, part, Nf, V, ep); break;
    case 2: launch_sym_on<2, EPI_STORE>(c, p, part, Nf, V, ep); break;
    case 3: launch_sym_on<3, EPI_STORE>(c, p, part, Nf, V, ep); break;
    case 4: launch_sym_on<4, EPI_STORE>(c, p, part, Nf, V, ep); break;
    case 5: launch_sym_on<5, EPI_STORE>(c, p, part, Nf, V, ep); break;
    default: throw Error(XM_EINVAL, "symmetric product supports r ≤ 5");
  }
}

void sym_plan_slot_destroy(void*& slot) {
  delete static_cast<SymPlan*>(slot);
  slot = nullptr;
}

template <int MODE>
static void sym_mode(xm_ctx* c, const double* V, int r, const SpmmEpiArgs& ep) {
  switch (r) {
    case 1: launch_sym<1, MODE>(c, V, ep); break;
    case 2: launch_sym<2, MODE>(c, V, ep); break;
    case 3: launch_sym<3, MODE>(c, V, ep); break;
    case 4: launch_sym<4, MODE>(c, V, ep); break;
    case 5: launch_sym<5, MODE>(c, V, ep); break;
    default: throw Error(XM_EINVAL, "symmetric SpMM supports r ≤ 5");
  }
}

void spmm_sym_launch(xm_ctx* c, const double* V, int r, int mode, const SpmmEpiArgs& ep) {
  switch (mode) {
    case EPI_STORE: sym_mode<EPI_STORE>(c, V, r, ep); break;
    case EPI_HVP: sym_mode<EPI_HVP>(c, V, r, ep); break;
    case EPI_ZMUL: sym_mode<EPI_ZMUL>(c, V, r, ep); break;
    case EPI_DF: sym_mode<EPI_DF>(c, V, r, ep); break;
    case EPI_GRAD: sym_mode<EPI_GRAD>(c, V, r, ep); break;
    default: throw Error(XM_EINVAL, "bad epilogue");
  }
}

}  // namespace xm
