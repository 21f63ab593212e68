// spmm_sym.cu — H6 with symmetric Q: out = Q·V streaming only the lower
// triangle (Q = Qᵀ by construction, Prop. 1) — half the HBM bytes of the
// full-row kernel (spmm.cu).
//
//   out_i = Σ_{j ≤ i} Q_ij V_j  +  Σ_{j > i} Q_ji V_j
//         = row part (lower triangle) + column part (strictly lower triangle)
//
// Geometry.  Units are the lower-triangular 128-row × 256-column blocks
// (I, J), J ≤ ⌊I/2⌋; a unit is 8 tiles of 16 rows × 256 columns (32 KB).  The
// W = 16·U tiles are split stream-K style into G = 148 equal contiguous ranges
// (one persistent CTA per SM), so every SM streams the same number of tiles.
// A CTA's range is a sequence of *segments* (maximal runs of tiles of one
// unit); a unit cut between two CTAs simply yields two segments.
//
// Per tile (warp w ↔ rows w, w+8; lane ℓ ↔ the 8 columns {2ℓ+64m, 2ℓ+64m+1},
// m = 0..3 — conflict-free LDS.128):
//   row part   r_i += Σ_j Q_ij V_j  with V_J for the lane's columns held in
//              registers for the whole segment; one 5-level shuffle reduction
//              per row, then lane 0 writes rowpart[u][ℓ] (each row of a unit
//              lives in exactly one tile ⇒ single writer);
//   column part c_j += Q_ij V_i (j < i), accumulated in registers over the
//              segment's rows (V_i broadcast from shared memory), then summed
//              over the 8 warps in a fixed order and written to colpart[segment].
// The producer thread streams each tile with ONE 2-D tensor TMA copy
// (cp.async.bulk.tensor.2d, L2 evict-first; rows / columns past n zero-filled)
// into a 5-stage ring (5 × 32 KB); the per-segment V_J / V_I blocks go through
// a 2-slot ring (1-D bulk copies).
//
// After a software grid barrier the same CTAs sum, in a fixed order, the row
// parts of units (K, 0..⌊K/2⌋) and the column parts of every segment of column
// block ⌊row/256⌋, and apply the per-camera epilogue (same modes as spmm.cu).
// Deterministic; algorithmic bytes per product: 8·n(n+1)/2 + 16·n·r.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "frame_ops.cuh"

#include <map>
#include <type_traits>

namespace xm {

namespace {
constexpr int kWarps = 8;
constexpr int kThreads = 32 * (kWarps + 1);
constexpr int BR = 128;                 // unit rows
constexpr int BC = 256;                 // unit columns
constexpr int TR = 16;                  // rows per tile (two per warp)
constexpr int kTilesPerUnit = BR / TR;  // 8
constexpr int kTileBytes = TR * BC * 8;  // 32 KB

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
// unit u → (I, J) using unit_base[I] = Σ_{I'<I} (⌊I'·BR/BC⌋ + 1)
__device__ __forceinline__ void unit_ij(int u, const int* __restrict__ ubase, int TRb, int& I, int& J) {
  int lo = 0, hi = TRb - 1;
  while (lo < hi) {  // largest I with ubase[I] ≤ u
    int mid = (lo + hi + 1) >> 1;
    if (ubase[mid] <= u) lo = mid; else hi = mid - 1;
  }
  I = lo;
  J = u - ubase[lo];
}
}  // namespace

// Static work plan for one (n, G): unit bases, per-CTA segment bases and the
// per-column-block list of segments (fixed summation order for the finish).
struct SymPlan {
  int n = 0, G = 0, TRb = 0, TCb = 0, U = 0, S = 0;
  const void* qptr = nullptr;  // Q the tensor map was encoded for
  int64_t ldq = 0;
  CUtensorMap tmq;
  DBuf<int> ubase;     // TRb + 1
  DBuf<int> segbase;   // G + 1
  DBuf<int> segunit;   // S
  DBuf<int> colptr;    // TCb + 1
  DBuf<int> colidx;    // S (segments grouped by column block, ordered by unit then CTA)
};

static SymPlan& sym_plan(xm_ctx* c) {
  if (!c->sym_plan) c->sym_plan = new SymPlan();
  SymPlan& p = *static_cast<SymPlan*>(c->sym_plan);
  int sms = 148;
  XM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const int n = c->n, G = std::min(148, sms);
  if (p.n == n && p.G == G && p.ubase.p && p.qptr == c->Q.p && p.ldq == c->ldq) return p;
  // Q tensor map: dims {n columns, n rows}, row pitch ldq·8 B, box TR × BC,
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
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)c->ldq * 8};
    cuuint32_t box[2] = {(cuuint32_t)BC, (cuuint32_t)TR};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&p.tmq, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, c->Q.p, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(XM_ECUDA, "cuTensorMapEncodeTiled failed");
    p.qptr = c->Q.p;
    p.ldq = c->ldq;
  }
  if (p.n == n && p.G == G && p.ubase.p) return p;
  p.n = n;
  p.G = G;
  p.TRb = ceil_div(n, BR);
  p.TCb = ceil_div(n, BC);
  std::vector<int> ub(p.TRb + 1, 0);
  for (int I = 0; I < p.TRb; ++I) ub[I + 1] = ub[I] + (I * BR) / BC + 1;
  p.U = ub[p.TRb];
  const int64_t W = (int64_t)p.U * kTilesPerUnit;
  std::vector<int> segbase(G + 1, 0), segunit;
  for (int cta = 0; cta < G; ++cta) {
    int64_t t0 = (int64_t)cta * W / G, t1 = (int64_t)(cta + 1) * W / G;
    segbase[cta] = (int)segunit.size();
    int last = -1;
    for (int64_t t = t0; t < t1; ++t) {
      int u = (int)(t / kTilesPerUnit);
      if (u != last) {
        segunit.push_back(u);
        last = u;
      }
    }
  }
  segbase[G] = (int)segunit.size();
  p.S = (int)segunit.size();
  auto unitJ = [&](int u) {
    int I = 0;
    while (ub[I + 1] <= u) ++I;
    return u - ub[I];
  };
  std::vector<std::vector<int>> bycol(p.TCb);
  for (int s = 0; s < p.S; ++s) bycol[unitJ(segunit[s])].push_back(s);  // s increasing ⇒ unit, then CTA order
  std::vector<int> colptr(p.TCb + 1, 0), colidx;
  for (int J = 0; J < p.TCb; ++J) {
    for (int s : bycol[J]) colidx.push_back(s);
    colptr[J + 1] = (int)colidx.size();
  }
  p.ubase.alloc(ub.size());
  p.segbase.alloc(segbase.size());
  p.segunit.alloc(std::max<size_t>(1, segunit.size()));
  p.colptr.alloc(colptr.size());
  p.colidx.alloc(std::max<size_t>(1, colidx.size()));
  XM_CUDA(cudaMemcpy(p.ubase.p, ub.data(), ub.size() * 4, cudaMemcpyHostToDevice));
  XM_CUDA(cudaMemcpy(p.segbase.p, segbase.data(), segbase.size() * 4, cudaMemcpyHostToDevice));
  if (!segunit.empty())
    XM_CUDA(cudaMemcpy(p.segunit.p, segunit.data(), segunit.size() * 4, cudaMemcpyHostToDevice));
  XM_CUDA(cudaMemcpy(p.colptr.p, colptr.data(), colptr.size() * 4, cudaMemcpyHostToDevice));
  if (!colidx.empty())
    XM_CUDA(cudaMemcpy(p.colidx.p, colidx.data(), colidx.size() * 4, cudaMemcpyHostToDevice));
  return p;
}

template <int R>
struct SymCfg {
  static constexpr int kVJ = BC * R;   // doubles
  static constexpr int kVI = BR * R;
  static constexpr int kStages = (R <= 3) ? 5 : 4;
  static constexpr size_t kSmem = (size_t)kStages * kTileBytes + 2 * (size_t)(kVJ + kVI) * 8 +
                                  4 * (size_t)BC * R * 8 + 64 * 8;
};

template <int R, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_spmm_sym(
    const __grid_constant__ CUtensorMap tmq, int N, int n, int TRb, int U,
    const int* __restrict__ ubase, const int* __restrict__ segbase, const int* __restrict__ colptr,
    const int* __restrict__ colidx, const double* __restrict__ V, double* __restrict__ rowpart,
    double* __restrict__ colpart, GridBar* __restrict__ gbar, SpmmEpiArgs ep) {
  using Cfg = SymCfg<R>;
  constexpr int kStages = Cfg::kStages;
  if (ep.stop && *ep.stop) return;
  if (ep.exec && blockIdx.x == 0 && threadIdx.x == 0) *ep.exec = 1;
  extern __shared__ __align__(128) unsigned char sm[];
  double* tiles = reinterpret_cast<double*>(sm);
  double* vbuf = tiles + (size_t)kStages * TR * BC;  // 2 slots × (V_J, V_I)
  double* colred = vbuf + 2 * (Cfg::kVJ + Cfg::kVI);  // [4 slots][BC][R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(colred + 4 * BC * R);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* vfull = bars + 2 * kStages;
  uint64_t* vempty = vfull + 2;

  const int G = gridDim.x;
  const int64_t W = (int64_t)U * kTilesPerUnit;
  const int64_t t0 = (int64_t)blockIdx.x * W / G;
  const int64_t t1 = (int64_t)(blockIdx.x + 1) * W / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], kWarps);
    }
    for (int s = 0; s < 2; ++s) {
      bar_init(&vfull[s], 1);
      bar_init(&vempty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0 && t0 < t1) {
      const uint64_t pq = pol_first(), pv = pol_last();
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmq)) : "memory");
      int it = 0, seg = 0, cur_u = -1, I = 0, J = 0;
      for (int64_t t = t0; t < t1; ++t, ++it) {
        const int u = (int)(t / kTilesPerUnit);
        const int tl = (int)(t % kTilesPerUnit);
        if (u != cur_u) {  // new segment: locate the unit, stage V_J and V_I
          unit_ij(u, ubase, TRb, I, J);
          const int vs = seg & 1;
          bar_wait(&vempty[vs], (unsigned)(((seg >> 1) & 1) ^ 1));
          const int nj = min(BC, n - J * BC), ni = min(BR, n - I * BR);
          const unsigned bj = (unsigned)(((nj * R + 1) & ~1) * 8);
          const unsigned bi = (unsigned)(((ni * R + 1) & ~1) * 8);
          bar_expect(&vfull[vs], bj + bi);
          double* vj = vbuf + (size_t)vs * (Cfg::kVJ + Cfg::kVI);
          bulk_g2s(vj, V + (int64_t)J * BC * R, bj, &vfull[vs], pv);
          bulk_g2s(vj + Cfg::kVJ, V + (int64_t)I * BR * R, bi, &vfull[vs], pv);
          cur_u = u;
          ++seg;
        }
        const int s = it % kStages;
        bar_wait(&empty[s], (unsigned)(((it / kStages) & 1) ^ 1));
        bar_expect(&full[s], (unsigned)kTileBytes);
        tma_tile(tiles + (size_t)s * TR * BC, &tmq, J * BC, I * BR + tl * TR, &full[s], pq);
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    int it = 0, seg = 0, cur_u = -1;
    int I = 0, J = 0;
    bool dblk = false;
    double vr[8][R];      // V_J rows for the lane's 8 columns
    double colacc[8][R];  // column partials for the lane's 8 columns
    const double* vi = nullptr;
    int vs = 0;
    auto flush = [&](int slot_seg) {
      // fixed-order cross-warp sum of colacc: warps w and w+4 share slot w
      // (w stores, w+4 adds), then slots 0..3 are summed left to right
      double* cr = colred + (warp & 3) * BC * R;
      if (warp < 4) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int cc = 0; cc < R; ++cc) cr[(2 * lane + 64 * m + h) * R + cc] = colacc[2 * m + h][cc];
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kWarps) : "memory");
      if (warp >= 4) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int cc = 0; cc < R; ++cc) cr[(2 * lane + 64 * m + h) * R + cc] += colacc[2 * m + h][cc];
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kWarps) : "memory");
      double* dst = colpart + ((int64_t)(segbase[blockIdx.x] + slot_seg)) * BC * R;
      for (int e = threadIdx.x; e < BC * R; e += 32 * kWarps)
        dst[e] = ((colred[e] + colred[BC * R + e]) + colred[2 * BC * R + e]) + colred[3 * BC * R + e];
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kWarps) : "memory");
    };
    // one row of a tile: row part (j ≤ jmax) and column part (j < i)
    auto do_row = [&](auto diag_tag, const double* st, int rl, int i, int64_t u) {
      constexpr bool DIAG = decltype(diag_tag)::value;
      double rs[R];
#pragma unroll
      for (int cc = 0; cc < R; ++cc) rs[cc] = 0.0;
      double vrow[R];
#pragma unroll
      for (int cc = 0; cc < R; ++cc) vrow[cc] = vi[rl * R + cc];
      const int jmax = i - J * BC;  // diagonal column (DIAG only)
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int jl = 2 * lane + 64 * m;
        const double2 q2 = *reinterpret_cast<const double2*>(st + jl);
        double qa = q2.x, qb = q2.y, ca = qa, cb = qb;
        if (DIAG) {  // row part j ≤ i, column part j < i; beyond: zero
          qa = (jl <= jmax) ? qa : 0.0;
          qb = (jl + 1 <= jmax) ? qb : 0.0;
          ca = (jl < jmax) ? q2.x : 0.0;
          cb = (jl + 1 < jmax) ? q2.y : 0.0;
        }
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
          rs[cc] = fma(qa, vr[2 * m][cc], fma(qb, vr[2 * m + 1][cc], rs[cc]));
          colacc[2 * m][cc] = fma(ca, vrow[cc], colacc[2 * m][cc]);
          colacc[2 * m + 1][cc] = fma(cb, vrow[cc], colacc[2 * m + 1][cc]);
        }
      }
#pragma unroll
      for (int cc = 0; cc < R; ++cc) {
        double v = rs[cc];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        rs[cc] = v;
      }
      if (lane == 0) {
        double* pr = rowpart + (u * BR + rl) * R;
#pragma unroll
        for (int cc = 0; cc < R; ++cc) pr[cc] = rs[cc];
      }
    };
    for (int64_t t = t0; t < t1; ++t, ++it) {
      const int u = (int)(t / kTilesPerUnit);
      const int tl = (int)(t % kTilesPerUnit);
      if (u != cur_u) {
        if (cur_u >= 0) {
          if (lane == 0) bar_arrive(&vempty[vs]);
          flush(seg - 1);
        }
        unit_ij(u, ubase, TRb, I, J);
        dblk = (J == (I * BR) / BC);
        vs = seg & 1;
        bar_wait(&vfull[vs], (unsigned)((seg >> 1) & 1));
        const double* vj = vbuf + (size_t)vs * (Cfg::kVJ + Cfg::kVI);
        vi = vj + Cfg::kVJ;
        const int nj = min(BC, n - J * BC);
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jl = 2 * lane + 64 * m + h;
#pragma unroll
            for (int cc = 0; cc < R; ++cc) {
              vr[2 * m + h][cc] = (jl < nj) ? vj[jl * R + cc] : 0.0;
              colacc[2 * m + h][cc] = 0.0;
            }
          }
        cur_u = u;
        ++seg;
      }
      const int s = it % kStages;
      bar_wait(&full[s], (unsigned)((it / kStages) & 1));
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const double* st = tiles + (size_t)s * TR * BC + (warp + 8 * half) * BC;
        const int rl = tl * TR + warp + 8 * half;  // row within the unit
        const int i = I * BR + rl;
#ifndef XM_EXP_NOCOMPUTE
        if (i < n) {
          if (dblk) do_row(std::true_type{}, st, rl, i, (int64_t)u);
          else do_row(std::false_type{}, st, rl, i, (int64_t)u);
        }
#else
        (void)st; (void)i;
#endif
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[s]);
    }
    if (cur_u >= 0) {
      if (lane == 0) bar_arrive(&vempty[vs]);
      flush(seg - 1);
    }
  }

  // ------------------------------------------------------------ finish (fused)
  // All row / column partials are published; CTA c now sums the partial lists
  // of the rows of frames [c·N/G, (c+1)·N/G) (warp per row, lanes split the
  // list, fixed xor-shuffle tree) and applies the per-camera epilogue.
#ifdef XM_EXP_NOFINISH
  return;
#endif
  grid_barrier(gbar, G);
  const int fa = (int)((int64_t)blockIdx.x * N / G), fb = (int)((int64_t)(blockIdx.x + 1) * N / G);
  double* qrow = tiles;  // pipeline smem is free now: [rows][R]
  for (int rr = warp; rr < 3 * (fb - fa); rr += kWarps + 1) {
    const int row = 3 * fa + rr;
    const int K = row / BR, l = row % BR;
    const int u0 = ubase[K], nu = ubase[K + 1] - u0;
    const int Jc = row / BC, m = row % BC;
    const int c0 = colptr[Jc], nc = colptr[Jc + 1] - c0;
    double acc[R];
#pragma unroll
    for (int cc = 0; cc < R; ++cc) acc[cc] = 0.0;
    for (int q = lane; q < nu + nc; q += 32) {
      const double* p = (q < nu) ? rowpart + ((int64_t)(u0 + q) * BR + l) * R
                                 : colpart + ((int64_t)colidx[c0 + q - nu] * BC + m) * R;
#pragma unroll
      for (int cc = 0; cc < R; ++cc) acc[cc] += p[cc];
    }
#pragma unroll
    for (int cc = 0; cc < R; ++cc) {
      double v = acc[cc];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) qrow[rr * R + cc] = v;
    }
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
// Kernel choice per (N, r), from tools/exp_sym.sh on B200:
//   B (N=2000): sym 41.4 µs vs full-row 51.1 µs at r=1, 57.9 vs 55.3 at r=3;
//   E (N=10155): sym 988 µs vs full-row 1033 µs at r=3.
// The fused finish + per-tile 2-sided update cost ~25 µs at N=2000, so the
// half-traffic kernel only pays for r = 1 (Lanczos) or once Q is large.
void sym_plan_destroy(xm_ctx* c) {
  delete static_cast<SymPlan*>(c->sym_plan);
  c->sym_plan = nullptr;
}

bool spmm_sym_supported(xm_ctx* c, int r) {
  if (c->world != 1 || r < 1 || r > 5 || c->opt.spmm_kernel == 1) return false;
  return c->opt.spmm_kernel == 2 || r == 1 || c->N >= 4000;
}

int spmm_sym_partials(xm_ctx* c) { return sym_plan(c).G; }

template <int R, int MODE>
static void launch_sym(xm_ctx* c, const double* V, const SpmmEpiArgs& ep) {
  SymPlan& p = sym_plan(c);
  // sized for the largest supported r once, so the address never changes when
  // the staircase climbs (the tCG graphs of lower ranks captured it)
  constexpr int kRmax = 5;
  const size_t rp = (size_t)p.U * BR * R;
  c->sym_part.alloc((size_t)p.U * BR * kRmax + (size_t)std::max(p.S, 1) * BC * kRmax + 64);
  double* rowpart = c->sym_part.p;
  double* colpart = c->sym_part.p + rp;
  if (!c->gbar.p) {
    c->gbar.alloc(4);
    XM_CUDA(cudaMemset(c->gbar.p, 0, 4 * sizeof(int)));
  }
  const size_t smem = SymCfg<R>::kSmem;
  static bool attr = false;
  if (!attr) {
    XM_CUDA(cudaFuncSetAttribute(k_spmm_sym<R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int nb = 0;
    XM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_spmm_sym<R, MODE>, kThreads, smem));
    if (nb < 1) throw Error(XM_ECUDA, "symmetric SpMM does not fit on an SM");
    attr = true;
  }
  k_spmm_sym<R, MODE><<<p.G, kThreads, smem, c->stream>>>(
      p.tmq, c->N, c->n, p.TRb, p.U, p.ubase.p, p.segbase.p, p.colptr.p, p.colidx.p, V, rowpart,
      colpart, reinterpret_cast<GridBar*>(c->gbar.p), ep);
  XM_CHECK_LAUNCH();
  count_launch(c, 1);
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
