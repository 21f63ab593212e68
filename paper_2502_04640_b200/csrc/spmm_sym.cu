// spmm_sym.cu — H6 with symmetric Q: out = Q·V streaming only the lower
// triangle (Q = Qᵀ by construction, Prop. 1), i.e. half of the HBM bytes of
// the full-row kernel.
//
//   out_i = Σ_{j ≤ i} Q_ij V_j  +  Σ_{j > i} Q_ji V_j
//         = (row part of the lower triangle) + (column part of the strictly lower triangle)
//
// Work units are the T(T+1)/2 lower-triangular 128×128 blocks (I, J ≥ ... J ≤ I),
// distributed as contiguous ranges over G = 148 persistent CTAs (one per SM).
// For unit (I, J) a CTA produces, deterministically,
//   rowpart[u][ℓ] = Σ_{j in block J, j ≤ i} Q_ij V_j      (ℓ = row within block I)
//   colpart[u][m] = Σ_{i in block I, i > j} Q_ij V_i      (m = column within block J)
// and k_sym_finish sums, for each output row in block K, the row parts of
// units (K, 0..K) and the column parts of units (K..T−1, K) in a fixed order,
// then applies the per-camera epilogue (same modes as spmm.cu).
//
// Pipeline per CTA: one producer thread streams 32-row × 128-column Q tiles
// (one cp.async.bulk per row, diagonal rows only up to the diagonal; L2
// evict-first) into a 4-stage ring, and per unit the V_J / V_I row blocks into
// a 2-slot ring.  8 consumer warps: warp w owns 4 rows of every tile, lane ℓ
// owns the 4 interleaved columns {2ℓ, 2ℓ+1, 64+2ℓ, 65+2ℓ} (conflict-free
// LDS.128).  V_J for the lane's columns lives in registers for the unit; the
// column partials accumulate in registers over the unit's 128 rows and are
// combined across warps in a fixed order through shared memory.
//
// Algorithmic bytes per product: 8·n(n+1)/2 (lower triangle of Q) + 16·n·r.
#include "frame_ops.cuh"

namespace xm {

namespace {
constexpr int kWarps = 8;
constexpr int kThreads = 32 * (kWarps + 1);
constexpr int BT = 128;          // unit block size
constexpr int TR = 32;           // rows per streamed tile
constexpr int kTiles = BT / TR;  // tiles per unit
constexpr int kStages = 4;
constexpr int kTileBytes = TR * BT * 8;  // 32 KB

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
__device__ __forceinline__ void unit_ij(int64_t u, int& I, int& J) {
  int i = (int)((sqrt(8.0 * (double)u + 1.0) - 1.0) * 0.5);
  while ((int64_t)(i + 1) * (i + 2) / 2 <= u) ++i;
  while ((int64_t)i * (i + 1) / 2 > u) --i;
  I = i;
  J = (int)(u - (int64_t)i * (i + 1) / 2);
}
}  // namespace

template <int R>
struct SymCfg {
  static constexpr int kVBlockBytes = BT * R * 8;           // one V row block
  static constexpr int kColRedBytes = kWarps * BT * R * 8;  // cross-warp column reduction
  static constexpr size_t kSmem = (size_t)kStages * kTileBytes + 2 * 2 * kVBlockBytes +
                                  kColRedBytes + 64 * 8;
};

template <int R>
__global__ void __launch_bounds__(kThreads, 1) k_spmm_sym(const double* __restrict__ Q, int64_t ldq,
                                                          int n, int T, const double* __restrict__ V,
                                                          double* __restrict__ part,
                                                          const int* __restrict__ stop,
                                                          int* __restrict__ exec) {
  using Cfg = SymCfg<R>;
  if (stop && *stop) return;
  if (exec && blockIdx.x == 0 && threadIdx.x == 0) *exec = 1;
  extern __shared__ __align__(128) unsigned char sm[];
  double* tiles = reinterpret_cast<double*>(sm);
  double* vbuf = reinterpret_cast<double*>(sm + (size_t)kStages * kTileBytes);  // [2 slots][VJ, VI]
  double* colred = vbuf + 2 * 2 * BT * R;                                           // [warp][BT][R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(colred + kWarps * BT * R);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* vfull = bars + 2 * kStages;
  uint64_t* vempty = vfull + 2;

  const int64_t U = (int64_t)T * (T + 1) / 2;
  const int64_t u0 = (int64_t)blockIdx.x * U / gridDim.x;
  const int64_t u1 = (int64_t)(blockIdx.x + 1) * U / gridDim.x;
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
    if (lane != 0) return;
    const uint64_t pq = pol_first(), pv = pol_last();
    int it = 0;
    int uu = 0;
    for (int64_t u = u0; u < u1; ++u, ++uu) {
      int I, J;
      unit_ij(u, I, J);
      const int vs = uu & 1;
      bar_wait(&vempty[vs], (unsigned)(((uu >> 1) & 1) ^ 1));
      const int nj = min(BT, n - J * BT), ni = min(BT, n - I * BT);
      const unsigned bj = (unsigned)(((nj * R + 1) & ~1) * 8), bi = (unsigned)(((ni * R + 1) & ~1) * 8);
      bar_expect(&vfull[vs], bj + bi);
      double* vj = vbuf + (size_t)vs * 2 * BT * R;
      bulk_g2s(vj, V + (int64_t)J * BT * R, bj, &vfull[vs], pv);
      bulk_g2s(vj + BT * R, V + (int64_t)I * BT * R, bi, &vfull[vs], pv);
      for (int t = 0; t < kTiles; ++t, ++it) {
        const int s = it % kStages;
        bar_wait(&empty[s], (unsigned)(((it / kStages) & 1) ^ 1));
        const int r0 = I * BT + t * TR;
        const int rows = max(0, min(TR, n - r0));
        unsigned total = 0;
        unsigned len[TR];
        for (int q = 0; q < rows; ++q) {
          int i = r0 + q;
          int cols = (I == J) ? (i - J * BT + 1) : nj;
          len[q] = (unsigned)(((cols + 1) & ~1) * 8);
          total += len[q];
        }
        bar_expect(&full[s], total);
        double* st = tiles + (size_t)s * TR * BT;
        for (int q = 0; q < rows; ++q)
          bulk_g2s(st + q * BT, Q + (int64_t)(r0 + q) * ldq + (int64_t)J * BT, len[q], &full[s], pq);
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  int it = 0;
  int uu = 0;
  const int c0 = 2 * lane, c1 = 64 + 2 * lane;  // lane's column pairs within the block
  for (int64_t u = u0; u < u1; ++u, ++uu) {
    int I, J;
    unit_ij(u, I, J);
    const bool diag = (I == J);
    const int vs = uu & 1;
    bar_wait(&vfull[vs], (unsigned)((uu >> 1) & 1));
    const double* vj = vbuf + (size_t)vs * 2 * BT * R;
    const double* vi = vj + BT * R;
    const int nj = min(BT, n - J * BT);
    double vr[4][R];  // V_J for the lane's 4 columns
    const int cl[4] = {c0, c0 + 1, c1, c1 + 1};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) vr[k][cc] = (cl[k] < nj) ? vj[cl[k] * R + cc] : 0.0;
    double colacc[4][R];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) colacc[k][cc] = 0.0;
    for (int t = 0; t < kTiles; ++t, ++it) {
      const int s = it % kStages;
      bar_wait(&full[s], (unsigned)((it / kStages) & 1));
      const double* st = tiles + (size_t)s * TR * BT;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rl = t * TR + warp * 4 + q;  // row within block I
        const int i = I * BT + rl;
        double rs[R];
#pragma unroll
        for (int cc = 0; cc < R; ++cc) rs[cc] = 0.0;
        if (i < n) {
          const double2 qa = *reinterpret_cast<const double2*>(st + (warp * 4 + q) * BT + c0);
          const double2 qb = *reinterpret_cast<const double2*>(st + (warp * 4 + q) * BT + c1);
          const double qv[4] = {qa.x, qa.y, qb.x, qb.y};
          double vrow[R];
#pragma unroll
          for (int cc = 0; cc < R; ++cc) vrow[cc] = vi[rl * R + cc];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int jl = cl[k];
            const bool in_row = diag ? (jl <= rl) : (jl < nj);
            const bool in_col = diag ? (jl < rl) : (jl < nj);
            const double x = in_row ? qv[k] : 0.0;
            const double y = in_col ? qv[k] : 0.0;
#pragma unroll
            for (int cc = 0; cc < R; ++cc) {
              rs[cc] = fma(x, vr[k][cc], rs[cc]);
              colacc[k][cc] = fma(y, vrow[cc], colacc[k][cc]);
            }
          }
        }
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
          double v = rs[cc];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          rs[cc] = v;
        }
        if (lane == 0 && i < n) {
          double* pr = part + (u * 2 * BT + rl) * R;
#pragma unroll
          for (int cc = 0; cc < R; ++cc) pr[cc] = rs[cc];
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[s]);
    }
    if (lane == 0) bar_arrive(&vempty[vs]);
    // column partials: registers → smem [warp][col][R] → fixed-order sum over warps
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) colred[(warp * BT + cl[k]) * R + cc] = colacc[k][cc];
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kWarps) : "memory");
    for (int e = threadIdx.x; e < nj * R; e += 32 * kWarps) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) sum += colred[w * BT * R + e];
      part[(u * 2 * BT + BT) * R + e] = sum;
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kWarps) : "memory");
  }
}

// ---------------------------------------------------------------- finish + epilogue
template <int R, int MODE>
__global__ void __launch_bounds__(128) k_sym_finish(int N, int n, int T, const double* __restrict__ part,
                                                    const double* __restrict__ V, SpmmEpiArgs ep) {
  if (ep.stop && *ep.stop) return;
  const int i = blockIdx.x * 128 + threadIdx.x;
  constexpr int NC = (MODE == EPI_GRAD) ? 3 : (MODE == EPI_DF ? 2 : 1);
  double pt[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) pt[q] = (MODE == EPI_GRAD && q == 2) ? 1.0e300 : 0.0;
  if (i < N) {
    Blk<R> qv;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int row = 3 * i + a;
      const int K = row / BT, l = row % BT;
      double acc[R];
#pragma unroll
      for (int cc = 0; cc < R; ++cc) acc[cc] = 0.0;
      for (int J = 0; J <= K; ++J) {  // row parts of units (K, J)
        const int64_t u = (int64_t)K * (K + 1) / 2 + J;
        const double* p = part + (u * 2 * BT + l) * R;
#pragma unroll
        for (int cc = 0; cc < R; ++cc) acc[cc] += p[cc];
      }
      for (int Ib = K; Ib < T; ++Ib) {  // column parts of units (Ib, K)
        const int64_t u = (int64_t)Ib * (Ib + 1) / 2 + K;
        const double* p = part + (u * 2 * BT + BT + l) * R;
#pragma unroll
        for (int cc = 0; cc < R; ++cc) acc[cc] += p[cc];
      }
#pragma unroll
      for (int cc = 0; cc < R; ++cc) qv.v[a][cc] = acc[cc];
    }
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
  if (MODE != EPI_STORE) block_reduce_store<NC, 128>(pt, ep.partials, MODE == EPI_GRAD ? 4u : 0u);
}

// ---------------------------------------------------------------- host side
bool spmm_sym_supported(xm_ctx* c, int r) { return c->world == 1 && r >= 1 && r <= 6 && c->use_sym; }

int spmm_sym_partials(xm_ctx* c) { return ceil_div(c->N, 128); }

template <int R, int MODE>
static void launch_sym(xm_ctx* c, const double* V, const SpmmEpiArgs& ep) {
  const int T = ceil_div(c->n, BT);
  const int64_t U = (int64_t)T * (T + 1) / 2;
  c->sym_part.alloc((size_t)U * 2 * BT * R + 64);
  const size_t smem = SymCfg<R>::kSmem;
  static bool attr = false;
  if (!attr) {
    XM_CUDA(cudaFuncSetAttribute(k_spmm_sym<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int G = (int)std::min<int64_t>(148, U);
  k_spmm_sym<R><<<G, kThreads, smem, c->stream>>>(c->Q.p, c->ldq, c->n, T, V, c->sym_part.p, ep.stop,
                                                  ep.exec);
  XM_CHECK_LAUNCH();
  k_sym_finish<R, MODE><<<ceil_div(c->N, 128), 128, 0, c->stream>>>(c->N, c->n, T, c->sym_part.p, V, ep);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
}

template <int MODE>
static void sym_mode(xm_ctx* c, const double* V, int r, const SpmmEpiArgs& ep) {
  switch (r) {
    case 1: launch_sym<1, MODE>(c, V, ep); break;
    case 2: launch_sym<2, MODE>(c, V, ep); break;
    case 3: launch_sym<3, MODE>(c, V, ep); break;
    case 4: launch_sym<4, MODE>(c, V, ep); break;
    case 5: launch_sym<5, MODE>(c, V, ep); break;
    case 6: launch_sym<6, MODE>(c, V, ep); break;
    default: throw Error(XM_EINVAL, "symmetric SpMM supports r ≤ 6");
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
