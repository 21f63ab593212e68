// spmm.cu — H6: Q·V for the tall-skinny BM factor V ∈ ℝ^{n×r} (cost,
// gradient, every HVP of tCG, Δf, escapes, Lanczos with r = 1), with the
// per-camera epilogues H7/H8/H11 fused in.  The paper applies its dense Q with
// cuBLAS matrix-vector products; here one streaming kernel
// reads each Q byte exactly once per product.
//
// Roofline: HBM-bound.  Algorithmic bytes per product = 8·nrows·n (Q) +
// 8·n·r (V) + 8·nrows·r (out); 2·nrows·n·r flop ⇒ 0.25·r flop/B ≪ the fp64
// ridge (≈6 flop/B): tensor cores are irrelevant.
//
// Design (sm_100a), one persistent CTA per SM:
//  * CTA c owns the frame-aligned row range of frames [c·N_own/G, (c+1)·N_own/G)
//    over ALL columns ⇒ no split-K partials, every output row is final (and
//    identical for any number of ranks), and the per-camera epilogue runs in
//    the same kernel.  G = min(148, N_own) ⇒ balanced to within one camera.
//  * warp-specialised TMA pipeline: one elected producer thread streams tiles
//    of 8 Q rows × KC columns (one cp.async.bulk per row, L2 evict-first) plus
//    the matching V chunk (KC × r, contiguous) into a ring of S stages guarded
//    by full/empty mbarriers (transaction-count completion).  Bytes in flight =
//    S × stage bytes (≥ 128 KB per SM) independent of register pressure.
//  * 8 consumer warps: warp w owns columns [64w, 64w+64) of every tile and all 8
//    rows; a lane reads its 2 V values per column pair once (r LDS.128) and
//    reuses them for the 8 rows (8 LDS.128 of Q) ⇒ shared-memory traffic
//    ≈ (1 + r/8)× the Q stream.  Per-row partials stay in registers across the
//    K loop and are reduced once per row group (shuffles, then a fixed-order
//    cross-warp sum) into a per-row accumulator in shared memory.
//  * epilogues (one thread per camera of the CTA): STORE, HVP
//    (Hv = P(2Qv − 2Λv), ⟨v, Hv⟩), ZMUL (Zv = Qv − Λv, ⟨v, Zv⟩), DF (QD,
//    ⟨QY, D⟩, ⟨D, QD⟩), GRAD (QY, Λ, grad, f, ‖g‖², min α); scalar partials per
//    CTA, reduced in a fixed order by the consumer ⇒ deterministic.
#include "pipeline.cuh"

namespace xm {

constexpr int kConsumerWarps = 8;
constexpr int kSpmmThreads = 32 * (kConsumerWarps + 1);  // + 1 producer warp
constexpr int kTileRows = 8;
constexpr int kTileCols = 64 * kConsumerWarps;  // 512 columns per tile
#ifndef XM_SPMM_PREFETCH
#define XM_SPMM_PREFETCH 0  // measured: L2 prefetch ahead of the ring slows B by 15 %
#endif
constexpr int kSpmmPrefetch = XM_SPMM_PREFETCH;  // L2 prefetch distance (tiles)

template <int R>
struct SpmmCfg {
  static constexpr int kVBytes = kTileCols * R * 8;
  static constexpr int kQBytes = kTileRows * kTileCols * 8;  // 32 KB
  static constexpr int kStageBytes = kQBytes + kVBytes;
  static constexpr int kStages = (kStageBytes * 4 <= 176 * 1024) ? 4 : (kStageBytes * 3 <= 192 * 1024 ? 3 : 2);
};

// EPI_TCG: the rest of one Steihaug–Toint iteration after Hδ's Q·δ rows
// (H8 + H9, the same arithmetic as k_tcg_update + k_tcg_dir in manifold.cu),
// with two software grid barriers instead of two more launches.  Thread t
// owns camera f0g + t of this CTA (≤ kSpmmThreads cameras per CTA, checked on
// the host), so δ, Hδ, η, Hη, r and Y stay in registers across the barriers.
// Every CTA re-derives α, τ, β and the stop tests from the same partials in
// the same order ⇒ identical decisions everywhere; CTA 0 writes the state.
template <int R>
__device__ __forceinline__ void tcg_tail(int nf, int f0g, const SpmmEpiArgs& ep,
                                         const TcgState& s0, double part) {
  constexpr int NT = kSpmmThreads;
  const int t = threadIdx.x;
  const bool has = t < nf;
  const int i = f0g + t;
  double* __restrict__ dir = ep.out;
  Blk<R> y, dv, e, he, rr;
  double L[6];
  if (has) {
    load_blk<R>(ep.Y, i, y);
    load_blk<R>(dir, i, dv);
#pragma unroll
    for (int q = 0; q < 6; ++q) L[q] = ep.lam[6 * i + q];
    // ⟨δ, Hδ⟩ = ⟨δ, 2Qδ − 2Λδ⟩ (δ tangent, P self-adjoint): camera part −2⟨δ_i, Λ_iδ_i⟩
    Blk<R> zero{}, lamd;
    sub_lam<R>(zero, L, dv, 0.0, 1.0, lamd);  // −Λ_iδ_i
    part = fma(2.0, dotb<R>(dv, lamd), part);
    load_blk<R>(ep.eta, i, e);
    load_blk<R>(ep.Heta, i, he);
    load_blk<R>(ep.res, i, rr);
  }
  const double pc = block_sum_fixed<NT>(part);
  if (t == 0) ep.partials[blockIdx.x] = pc;
  XM_STAMP(2);
  grid_sync(ep.gsync, gridDim.x);
  XM_STAMP(3);
  // ---- α, e_Pe′, boundary / τ  (k_tcg_update)
  TcgState s = s0;
  const double dHd = block_sum_partials<NT>(ep.partials, gridDim.x);
  s.d_Hd = dHd;
  s.n_hvp += 1;
  const double alpha = (dHd != 0.0) ? s.z / dHd : INFINITY;
  const double e_new = s.e_Pe + 2.0 * alpha * s.e_Pd + alpha * alpha * s.d_Pd;
  const double D2 = s.Delta * s.Delta;
  s.alpha = alpha;
  s.e_Pe_new = e_new;
  if (dHd <= 0.0 || e_new >= D2) {
    s.tau = (-s.e_Pd + sqrt(s.e_Pd * s.e_Pd + s.d_Pd * (D2 - s.e_Pe))) / s.d_Pd;
    s.boundary = 1;
    s.stop = (dHd <= 0.0) ? TCG_NEGCURV : TCG_EXCEEDED;
  } else {
    s.boundary = 0;
  }
  const double a = s.boundary ? s.tau : alpha;
  double rn2 = 0.0;
  Blk<R> hd;
  if (has) {
    Blk<R> qv;  // this camera's Q·δ rows, written by whichever CTA streamed them
    const double* qp = ep.out2 + (int64_t)3 * i * R;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) qv.v[p][cc] = __ldcg(qp + p * R + cc);
    sub_lam<R>(qv, L, dv, 2.0, 2.0, hd);  // Hδ = P(2Qδ − 2Λδ)
    project_blk<R>(y, i == 0, hd);
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) {
        e.v[p][cc] = fma(a, dv.v[p][cc], e.v[p][cc]);
        he.v[p][cc] = fma(a, hd.v[p][cc], he.v[p][cc]);
      }
    store_blk<R>(ep.eta, i, e);
    store_blk<R>(ep.Heta, i, he);
    if (!s.boundary) {
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) rr.v[p][cc] = fma(a, hd.v[p][cc], rr.v[p][cc]);
      project_blk<R>(y, i == 0, rr);
      store_blk<R>(ep.res, i, rr);
      rn2 = frob2<R>(rr);
    }
  }
  if (s.boundary) {
    if (blockIdx.x == 0 && t == 0) *ep.st = s;
    return;
  }
  const double pr = block_sum_fixed<NT>(rn2);
  if (t == 0) ep.p2[blockIdx.x] = pr;
  XM_STAMP(4);
  grid_sync(ep.gsync, gridDim.x);
  XM_STAMP(5);
  // ---- stop tests, β, recurrences  (k_tcg_dir)
  const double z = block_sum_partials<NT>(ep.p2, gridDim.x);
  s.e_Pe = s.e_Pe_new;
  s.z_old = s.z;
  s.z = z;
  s.j += 1;
  if (sqrt(z) <= s.r0 * fmin(pow(s.r0, s.theta), s.kappa)) {
    s.stop = TCG_CONVERGED;
  } else {
    s.beta = s.z / s.z_old;
    s.e_Pd = s.beta * (s.e_Pd + s.alpha * s.d_Pd);
    s.d_Pd = s.z + s.beta * s.beta * s.d_Pd;
    if (s.j >= s.max_inner) s.stop = TCG_MAXINNER;
  }
  if (blockIdx.x == 0 && t == 0) *ep.st = s;
  if (s.stop || !has) return;
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int cc = 0; cc < R; ++cc) dv.v[p][cc] = fma(s.beta, dv.v[p][cc], -rr.v[p][cc]);
  store_blk<R>(dir, i, dv);  // δ ← −r + βδ (own cameras; every CTA is past its Q·δ)
  XM_STAMP(6);
}

template <int R, int MODE>
__global__ void __launch_bounds__(kSpmmThreads, 1) k_spmm(
    const double* __restrict__ Q, int64_t ldq, int n, int f_lo_rank, int nframes_own,
    const double* __restrict__ V, SpmmEpiArgs ep) {
  using Cfg = SpmmCfg<R>;
  constexpr int S = Cfg::kStages;
  if (ep.stop && *ep.stop) return;
  if (ep.exec && blockIdx.x == 0 && threadIdx.x == 0) *ep.exec = 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stage_base = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  double* red = reinterpret_cast<double*>(empty + S);   // [warps][kTileRows][R]
  double* acc = red + kConsumerWarps * kTileRows * R;   // [rows_cta][R]

  const int G = gridDim.x;
  // cameras [fa, fb) of this CTA (epilogues); Q rows [row_base, row_base + nrow):
  // the cameras' rows, or for EPI_TCG an even split of all rows (the camera
  // work runs after a grid barrier, so the stream need not be frame-aligned)
  const int fa = (int)((int64_t)blockIdx.x * nframes_own / G);
  const int fb = (int)((int64_t)(blockIdx.x + 1) * nframes_own / G);
  const int row_base = (MODE == EPI_TCG) ? (int)((int64_t)blockIdx.x * 3 * nframes_own / G) : 3 * fa;
  const int nrow = (MODE == EPI_TCG)
                       ? (int)((int64_t)(blockIdx.x + 1) * 3 * nframes_own / G) - row_base
                       : 3 * (fb - fa);
  const int ngroups = (nrow + kTileRows - 1) / kTileRows;
  const int nchunks = (n + kTileCols - 1) / kTileCols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int t = threadIdx.x; t < nrow * R; t += kSpmmThreads) acc[t] = 0.0;
  __shared__ TcgState ts0;  // EPI_TCG: the iteration's starting state (read before any write)
  if (MODE == EPI_TCG && threadIdx.x == 0) ts0 = *ep.st;
  if (MODE == EPI_TCG) XM_STAMP(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_v = policy_evict_last();
      // L2 prefetch kSpmmPrefetch tiles ahead of the smem ring: more HBM
      // requests in flight than the ring's S × 32 KB
      auto prefetch_tile = [&](int tp) {
        if (tp >= ngroups * nchunks) return;
        const int gp = tp / nchunks, jp = tp % nchunks;
        const int rp0 = gp * kTileRows, rowsp = min(kTileRows, nrow - rp0);
        const int kp0 = jp * kTileCols, klenp = min(kTileCols, n - kp0);
        for (int q = 0; q < rowsp; ++q)
          prefetch_l2(Q + (int64_t)(row_base + rp0 + q) * ldq + kp0,
                      (unsigned)(((klenp + 1) & ~1) * 8));
      };
      if (kSpmmPrefetch > 0)
        for (int tp = 0; tp < kSpmmPrefetch; ++tp) prefetch_tile(tp);
      int it = 0;
      for (int g = 0; g < ngroups; ++g) {
        const int r0 = g * kTileRows;
        const int rows = min(kTileRows, nrow - r0);
        for (int j = 0; j < nchunks; ++j, ++it) {
          const int s = it % S;
          const unsigned ph = (unsigned)((it / S) & 1);
          mbar_wait(&empty[s], ph ^ 1u);
          const int k0 = j * kTileCols;
          const int klen = min(kTileCols, n - k0);
          const unsigned qb = (unsigned)(((klen + 1) & ~1) * 8);  // 16-B multiple (pad ≤ 1 col)
          const unsigned vb = (unsigned)(((klen * R + 1) & ~1) * 8);
          mbar_expect_tx(&full[s], qb * rows + vb);
          double* st = stage_base + (size_t)s * (Cfg::kStageBytes / 8);
          for (int q = 0; q < rows; ++q)
            tma_load_1d(st + q * kTileCols, Q + (int64_t)(row_base + r0 + q) * ldq + k0, qb,
                        &full[s], pol_q);
          tma_load_1d(st + kTileRows * kTileCols, V + (int64_t)k0 * R, vb, &full[s], pol_v);
          if (kSpmmPrefetch > 0) prefetch_tile(it + kSpmmPrefetch);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    int it = 0;
    const int col = 64 * warp + 2 * lane;  // this lane's column pair within a tile
    for (int g = 0; g < ngroups; ++g) {
      const int r0 = g * kTileRows;
      const int rows = min(kTileRows, nrow - r0);
      double a[kTileRows][R];
#pragma unroll
      for (int q = 0; q < kTileRows; ++q)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) a[q][cc] = 0.0;
      for (int j = 0; j < nchunks; ++j, ++it) {
        const int s = it % S;
        const unsigned ph = (unsigned)((it / S) & 1);
        mbar_wait(&full[s], ph);
        const int klen = min(kTileCols, n - j * kTileCols);
        const double* st = stage_base + (size_t)s * (Cfg::kStageBytes / 8);
        const double* vs = st + kTileRows * kTileCols;
        if (col + 1 < klen) {
          double v0[R], v1[R];
#pragma unroll
          for (int cc = 0; cc < R; ++cc) {
            v0[cc] = vs[col * R + cc];
            v1[cc] = vs[(col + 1) * R + cc];
          }
#pragma unroll
          for (int q = 0; q < kTileRows; ++q) {
            if (q < rows) {
              double2 qv = *reinterpret_cast<const double2*>(st + q * kTileCols + col);
#pragma unroll
              for (int cc = 0; cc < R; ++cc) a[q][cc] = fma(qv.x, v0[cc], fma(qv.y, v1[cc], a[q][cc]));
            }
          }
        } else if (col < klen) {  // odd tail column
#pragma unroll
          for (int q = 0; q < kTileRows; ++q) {
            if (q < rows) {
              double qq = st[q * kTileCols + col];
#pragma unroll
              for (int cc = 0; cc < R; ++cc) a[q][cc] = fma(qq, vs[col * R + cc], a[q][cc]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // reduce the row group: lanes (shuffles) → warps (fixed order) → acc
#pragma unroll
      for (int q = 0; q < kTileRows; ++q)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
          double v = a[q][cc];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          a[q][cc] = v;
        }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kTileRows; ++q)
#pragma unroll
          for (int cc = 0; cc < R; ++cc) red[(warp * kTileRows + q) * R + cc] = a[q][cc];
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kConsumerWarps) : "memory");
      for (int t = threadIdx.x; t < rows * R; t += 32 * kConsumerWarps) {
        double sum = 0.0;
        for (int w = 0; w < kConsumerWarps; ++w) sum += red[w * kTileRows * R + t];
        acc[r0 * R + t] = sum;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kConsumerWarps) : "memory");
    }
  }
  __syncthreads();
  // ------------------------------------------------------------ epilogue
  const int f0g = f_lo_rank + fa;  // global frame index of the CTA's first frame
  if (MODE == EPI_STORE) {
    double* out = ep.out + (int64_t)(f_lo_rank * 3 + row_base) * R;
    for (int t = threadIdx.x; t < nrow * R; t += kSpmmThreads) out[t] = acc[t];
    return;
  }
  if constexpr (MODE == EPI_TCG) {
    XM_STAMP(1);
    // Q·δ rows → ep.out2 (read back by the owning cameras after the barrier),
    // and this CTA's rows' share of ⟨δ, 2Qδ⟩
    double part = 0.0;
    for (int t = threadIdx.x; t < nrow * R; t += kSpmmThreads) {
      const int64_t g = (int64_t)(f_lo_rank * 3 + row_base) * R + t;
      const double q = acc[t];
      ep.out2[g] = q;
      part = fma(2.0 * q, V[g], part);
    }
    tcg_tail<R>(fb - fa, f0g, ep, ts0, part);
    return;
  }
  constexpr int NC = (MODE == EPI_GRAD) ? 3 : (MODE == EPI_DF ? 2 : 1);
  double part[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) part[q] = (MODE == EPI_GRAD && q == 2) ? 1.0e300 : 0.0;
  for (int lf = threadIdx.x; lf < fb - fa; lf += kSpmmThreads) {
    const int i = f0g + lf;
    Blk<R> qv;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) qv.v[p][cc] = acc[(3 * lf + p) * R + cc];
    if (MODE == EPI_HVP) {
      Blk<R> y, vv, w;
      load_blk<R>(ep.Y, i, y);
      load_blk<R>(V, i, vv);
      double L[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) L[q] = ep.lam[6 * i + q];
      sub_lam<R>(qv, L, vv, 2.0, 2.0, w);  // 2Qv − 2Λv
      project_blk<R>(y, i == 0, w);
      store_blk<R>(ep.out2, i, w);
      part[0] += dotb<R>(vv, w);
    } else if (MODE == EPI_ZMUL) {
      Blk<R> vv, w;
      load_blk<R>(V, i, vv);
      double L[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) L[q] = ep.lam[6 * i + q];
      sub_lam<R>(qv, L, vv, 1.0, 1.0, w);  // Qv − Λv
      store_blk<R>(ep.out, i, w);
      part[0] += dotb<R>(vv, w);
    } else if (MODE == EPI_DF) {
      Blk<R> d, qy;
      load_blk<R>(V, i, d);
      load_blk<R>(ep.aux, i, qy);
      store_blk<R>(ep.out, i, qv);
      part[0] += dotb<R>(qy, d);
      part[1] += dotb<R>(d, qv);
    } else if (MODE == EPI_GRAD) {
      Blk<R> y, gr;
      load_blk<R>(V, i, y);  // V = Y
      store_blk<R>(ep.out, i, qv);
      double M[3][3], L[6];
      mul_abt<R>(qv, y, M);
      double alpha = frob2<R>(y) / 3.0;
      sym_lambda(M, i == 0, alpha, L);
#pragma unroll
      for (int q = 0; q < 6; ++q) ep.lam_out[6 * i + q] = L[q];
      sub_lam<R>(qv, L, y, 2.0, 2.0, gr);
      store_blk<R>(ep.out2, i, gr);
      part[0] += dotb<R>(y, qv);
      part[1] += frob2<R>(gr);
      if (i > 0) part[2] = fmin(part[2], alpha);
    }
  }
  // fixed-order reduction over the 9 warps: shuffles, then warp 0 in order
  __shared__ double wsum[kConsumerWarps + 1][NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    double v = part[q];
    const bool is_min = (MODE == EPI_GRAD && q == 2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_min ? fmin(v, u) : v + u;
    }
    if (lane == 0) wsum[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < NC) {
    const int q = threadIdx.x;
    const bool is_min = (MODE == EPI_GRAD && q == 2);
    double v = wsum[0][q];
    for (int w = 1; w <= kConsumerWarps; ++w) v = is_min ? fmin(v, wsum[w][q]) : v + wsum[w][q];
    ep.partials[blockIdx.x * NC + q] = v;
  }
}

// grid of the full-row kernel (k_spmm, every epilogue incl. EPI_TCG)
static int spmm_fullrow_grid(xm_ctx* c) {
  int nown = std::max(1, c->f1 - c->f0);
  return std::max(1, std::min(148, nown));
}
// grid (= number of per-CTA scalar partials) of a plain product at rank r
int spmm_grid(xm_ctx* c, int r) {
  if (spmm_sym_supported(c, r)) return spmm_sym_partials(c);
  return spmm_fullrow_grid(c);
}

template <int R, int MODE>
static void launch_r(xm_ctx* c, const double* V, const SpmmEpiArgs& ep) {
  using Cfg = SpmmCfg<R>;
  const int G = spmm_fullrow_grid(c);
  const int nown = c->f1 - c->f0;
  const int rows_max = 3 * ((nown + G - 1) / G);
  size_t smem = (size_t)Cfg::kStages * Cfg::kStageBytes + 2 * Cfg::kStages * 8 +
                (size_t)kConsumerWarps * kTileRows * R * 8 + (size_t)rows_max * R * 8;
  if (smem > 227 * 1024) throw Error(XM_EINVAL, "SpMM shared memory plan exceeds 227 KB");
  auto kern = k_spmm<R, MODE>;
  ensure_smem_attr((const void*)kern, smem);
  if (MODE == EPI_TCG) {
    // grid barriers inside: cooperative launch guarantees the G CTAs are co-resident
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kSpmmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    XM_CUDA(cudaLaunchKernelEx(&cfg, kern, (const double*)c->Q.p, (int64_t)c->ldq, c->n, c->f0,
                               nown, V, ep));
  } else {
    kern<<<G, kSpmmThreads, smem, c->stream>>>(c->Q.p, c->ldq, c->n, c->f0, nown, V, ep);
  }
  XM_CHECK_LAUNCH();
  count_launch(c);
}

template <int MODE>
static void launch_mode(xm_ctx* c, const double* V, int r, const SpmmEpiArgs& ep) {
  switch (r) {
#define XM_R(RR) case RR: launch_r<RR, MODE>(c, V, ep); break;
    XM_R(1) XM_R(2) XM_R(3) XM_R(4) XM_R(5) XM_R(6) XM_R(7) XM_R(8) XM_R(9) XM_R(10) XM_R(11)
    XM_R(12)
#undef XM_R
    default: throw Error(XM_EINVAL, "rank r out of range (1..12)");
  }
}

static void launch_tcg(xm_ctx* c, const double* V, int r, const SpmmEpiArgs& ep) {
  switch (r) {
#define XM_R(RR) case RR: launch_r<RR, EPI_TCG>(c, V, ep); break;
    XM_R(1) XM_R(2) XM_R(3) XM_R(4) XM_R(5) XM_R(6)
#undef XM_R
    default: throw Error(XM_EINVAL, "fused tCG supports r ≤ 6");
  }
}

bool tcg_fused_supported(xm_ctx* c, int r) {
  if (!c->fused_tcg || c->world != 1 || r < 1 || r > 6 || !tcg_fullrow_ok(c) || c->N < 1 ||
      !fused_epilogues(c))  // App. D terms / matrix-free products: unfused epilogues only
    return false;
  const int G = spmm_fullrow_grid(c);
  return ceil_div(c->N, G) <= kSpmmThreads;
}

// Algorithmic bytes of one product: Q (full rows, or the lower triangle when
// the symmetric kernel runs) + V in + result out.  The fused tCG iteration
// (EPI_TCG) instead moves Q + δ, then per camera reads Y, η, Hη, r, δ and
// writes η, Hη, r, δ (+ Λ): 8·n·n + 9·8·n·r + 48·N.
static double alg_bytes(xm_ctx* c, int r, int mode) {
  const double n = c->n;
  double qb;
  if (c->world > 1) {  // this rank's band: rows [a, b), columns ≤ row (lower trapezoid)
    const double a = c->row0, b = (double)c->row0 + c->nrows;
    qb = 8.0 * ((b * (b + 1) - a * (a + 1)) / 2);
    return qb + 8.0 * n * r + 8.0 * n * r;  // V in, the full-length partial out
  }
  qb = (mode != EPI_TCG && spmm_sym_supported(c, r)) ? 8.0 * n * (n + 1) / 2
                                                     : 8.0 * (double)c->nrows * n;
  if (mode == EPI_TCG) return qb + 9.0 * 8.0 * n * r + 48.0 * c->N;
  return qb + 8.0 * n * r + 8.0 * (double)c->nrows * r;
}

// Profiling (opt.profile): a CUDA event pair around one product on the
// library's stream plus an exec flag the product's first kernel sets when it
// really runs (graph replays past a tCG stop early-exit and are not counted);
// inside a graph capture the events and flag belong to the graph.
struct ProdTimer {
  cudaEvent_t e1 = nullptr;
  int* exec = nullptr;
};

static ProdTimer prod_timer_begin(xm_ctx* c, double bytes) {
  ProdTimer t;
  if (!c->opt.profile) return t;
  cudaEvent_t e0 = nullptr;
  if (c->cap_target) {
    auto* g = c->cap_target;
    size_t pair = g->bytes.size();
    if ((pair + 1) * sizeof(int) > g->execf.n * sizeof(int))
      throw Error(XM_EINVAL, "graph profiling slots exhausted");
    XM_CUDA(cudaEventCreate(&e0));
    XM_CUDA(cudaEventCreate(&t.e1));
    g->ev.push_back(e0);
    g->ev.push_back(t.e1);
    g->bytes.push_back(bytes);
    t.exec = g->execf.p + pair;
    // External ⇒ captured as an event-record node (plain records are capture markers)
    XM_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
  } else {
    if (c->ev_pool.empty()) {
      for (int q = 0; q < 1024; ++q) {
        cudaEvent_t e;
        XM_CUDA(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
      }
      c->ev_exec.alloc(512);
      c->ev_bytes.assign(512, 0.0);
      XM_CUDA(cudaMemsetAsync(c->ev_exec.p, 0, 512 * sizeof(int), c->stream));
    }
    if (c->ev_used + 2 > c->ev_pool.size()) harvest_events(c);
    e0 = c->ev_pool[c->ev_used++];
    t.e1 = c->ev_pool[c->ev_used++];
    size_t pair = c->ev_used / 2 - 1;
    t.exec = c->ev_exec.p + pair;
    c->ev_bytes[pair] = bytes;
    XM_CUDA(cudaEventRecord(e0, c->stream));
  }
  return t;
}

static void prod_timer_end(xm_ctx* c, const ProdTimer& t) {
  if (!t.e1) return;
  if (c->cap_target) XM_CUDA(cudaEventRecordWithFlags(t.e1, c->stream, cudaEventRecordExternal));
  else XM_CUDA(cudaEventRecord(t.e1, c->stream));
}

// One (optionally profiled) SpMM launch with epilogue `mode` on this rank's rows.
void spmm(xm_ctx* c, const double* V, int r, int mode, const SpmmEpiArgs& ep_in) {
  if (mode != EPI_STORE && c->world > 1)
    throw Error(XM_EINVAL, "fused epilogues need world == 1 (use spmm_full + epilogue kernels)");
  SpmmEpiArgs ep = ep_in;
  const ProdTimer tm = prod_timer_begin(c, alg_bytes(c, r, mode));
  if (tm.exec) ep.exec = tm.exec;
  if (mode != EPI_TCG && spmm_sym_supported(c, r)) {
    spmm_sym_launch(c, V, r, mode, ep);
  } else switch (mode) {
    case EPI_STORE: launch_mode<EPI_STORE>(c, V, r, ep); break;
    case EPI_HVP: launch_mode<EPI_HVP>(c, V, r, ep); break;
    case EPI_ZMUL: launch_mode<EPI_ZMUL>(c, V, r, ep); break;
    case EPI_DF: launch_mode<EPI_DF>(c, V, r, ep); break;
    case EPI_GRAD: launch_mode<EPI_GRAD>(c, V, r, ep); break;
    case EPI_TCG: launch_tcg(c, V, r, ep); break;
    default: throw Error(XM_EINVAL, "bad epilogue");
  }
  prod_timer_end(c, tm);
  c->stats.spmm_calls++;
  c->stats.spmm_rows = c->nrows;
}

__global__ void k_pack_cols(int64_t n, int r, int c0, int w, const double* __restrict__ V,
                            double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  const int64_t i = t / w;
  out[t] = V[i * r + c0 + (int)(t - i * w)];
}
__global__ void k_unpack_cols(int64_t n, int r, int c0, int w, const double* __restrict__ in,
                              double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  const int64_t i = t / w;
  out[i * r + c0 + (int)(t - i * w)] = in[t];
}

// Full product into out (replicated n × r).  One GPU: one launch.  world > 1
// (band layout, SURVEY §8(e) composed with the symmetric stream): every rank
// streams the lower trapezoid of its band with the lower-triangle kernel,
// which yields the band rows' row parts and the column parts of every row
// above (a full-length n × r partial, zero below the band); ONE all-reduce of
// those partials (n·r·8 bytes, ≈ 1 MB at E) replaces the all-gather of full-row
// shards and halves each rank's Q bytes.  r > 5: column groups of ≤ 5.
void spmm_full(xm_ctx* c, const double* V, int r, double* out_full, const int* stop) {
  if (c->implicit_active) {  // NEXT-1: matrix-free (implicit.cu); after a tCG stop the
    // passes of a graph replay early-exit, their result is ignored by the update kernels
    const ProdTimer tm = prod_timer_begin(c, implicit_alg_bytes(c, r));
    implicit_product(c, V, r, out_full, stop, tm.exec);
    prod_timer_end(c, tm);
    c->stats.spmm_calls++;
    return;
  }
  SpmmEpiArgs ep{};
  ep.stop = stop;
  if (c->world == 1 || r <= 5) {
    ep.out = out_full;
    spmm(c, V, r, EPI_STORE, ep);
  } else {
    const int64_t n = c->n;
    DBuf<double>& pv = scratch_f64(c, "band_pack_v");
    DBuf<double>& po = scratch_f64(c, "band_pack_o");
    pv.alloc((size_t)n * 5 + 64);
    po.alloc((size_t)n * 5 + 64);
    for (int c0 = 0; c0 < r; c0 += 5) {
      const int w = std::min(5, r - c0);
      k_pack_cols<<<ceil_div(n * w, 256), 256, 0, c->stream>>>(n, r, c0, w, V, pv.p);
      XM_CHECK_LAUNCH();
      ep.out = po.p;
      spmm(c, pv.p, w, EPI_STORE, ep);
      k_unpack_cols<<<ceil_div(n * w, 256), 256, 0, c->stream>>>(n, r, c0, w, po.p, out_full);
      XM_CHECK_LAUNCH();
      count_launch(c, 2);
    }
  }
  if (c->world > 1) nccl_allreduce_sum(c, out_full, (size_t)c->n * r);
}

// Accumulate the CUDA-event time of every profiled SpMM launch that actually
// ran (speculative launches that early-exited are skipped) into stats.
void harvest_events(xm_ctx* c) {
  if (c->ev_used == 0) return;
  XM_CUDA(cudaEventSynchronize(c->ev_pool[c->ev_used - 1]));
  std::vector<int> exec(c->ev_used / 2);
  XM_CUDA(cudaMemcpy(exec.data(), c->ev_exec.p, exec.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (size_t q = 0; q + 1 < c->ev_used; q += 2) {
    if (!exec[q / 2]) continue;
    float ms = 0.f;
    XM_CUDA(cudaEventElapsedTime(&ms, c->ev_pool[q], c->ev_pool[q + 1]));
    c->stats.spmm_ms += ms;
    c->stats.spmm_timed++;
    c->stats.spmm_alg_bytes += c->ev_bytes[q / 2];
  }
  XM_CUDA(cudaMemsetAsync(c->ev_exec.p, 0, 512 * sizeof(int), c->stream));
  c->ev_used = 0;
}

}  // namespace xm
