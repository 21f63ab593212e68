// tcg_persist.cu — H8 + H9: the whole Steihaug–Toint truncated-CG solve of
// one trust-region step (Manopt's tCG) in ONE
// persistent cooperative kernel, on one GPU with the full-row Q stream.
//
// Per iteration k (same arithmetic as k_tcg_update / k_tcg_dir, manifold.cu):
//   stream  Qδ_k for this CTA's rows (Q tiles by TMA, δ_k built on the fly)
//   ── grid barrier A ──  d_Hd = ⟨δ_k, Hδ_k⟩ → α, boundary / τ
//   cameras: Hδ = P(2Qδ − 2Λδ), η += αδ, Hη += αHδ, r += αHδ (projected)
//   ── grid barrier B ──  ‖r‖² → stop tests, β, δ_{k+1} = −r_{k+1} + βδ_k
//
// What the persistent form buys over one launch per iteration:
//  * no launch, no pipeline drain / fill between iterations — the Q producer
//    warp keeps prefetching the next iteration's Q tiles (Q never changes)
//    while the consumers are in the barrier / camera phases;
//  * no third barrier for δ: the next stream needs δ_{k+1} for ALL columns,
//    which consumers form on the fly from r_{k+1} and δ_k tiles (TMA-loaded
//    next to the Q tile) as −r + βδ with the same fma the owners use, so every
//    CTA sees bitwise the same δ; owners write δ_{k+1} into the other half of
//    a ping-pong pair for the stream after next.
//
// Tiling.  The L2 slices, not HBM, cap the stream when vector tiles are
// re-read per small row group (B200: ≈ 8.8 TB/s through L2 for Q + V traffic,
// measured).  So a tile is a whole ROW BLOCK of the CTA (≤ 48
// rows, one 1-D bulk copy per row) × 128 columns: each r / δ element is read
// from L2 once per row block instead of once per 8 rows.  8 consumer warps =
// 4 row quarters × 2 column halves; a lane owns 2 columns and ≤ 12 rows and
// reduces once per row block.  Rows are split evenly over the CTAs (the
// camera work follows barrier A and reads Qδ rows back from L2); cameras by
// ⌊N·c/G⌋ (≤ 256 per CTA).  Determinism: fixed-order partial sums, identical
// decisions in every CTA.
#include <cudaTypedefs.h>

#include "pipeline.cuh"

namespace xm {

namespace {
constexpr int kPW = 8;                  // consumer warps
constexpr int kPC = 32 * kPW;           // consumer threads
constexpr int kPThreads = kPC + 64;     // + two producer warps (Q tiles; r / δ tiles)
constexpr int kBlockRows = 48;          // rows per row block (4 quarters × ≤ 12)
constexpr int kQuarterRows = kBlockRows / 4;
constexpr int kPCols = 128;             // columns per tile (2 halves × 32 lanes × 2)


__device__ __forceinline__ void cbar() {  // consumers only (the producers keep streaming)
  asm volatile("bar.sync 1, %0;\n" ::"n"(kPC) : "memory");
}
// fixed-order sum over the 256 consumer threads; every consumer gets the value
__device__ __forceinline__ double csum(double v, double* ws) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  cbar();
  double t = ws[0];
#pragma unroll
  for (int w = 1; w < kPW; ++w) t += ws[w];
  cbar();
  return t;
}
__device__ __forceinline__ double csum_partials(const double* part, int n, double* ws) {
  double a = 0.0;
  for (int b = threadIdx.x; b < n; b += kPC) a += __ldcg(part + b);
  return csum(a, ws);
}
// grid barrier among the consumer groups of all CTAs (see grid_sync)
__device__ __forceinline__ void cgrid_sync(unsigned long long* cnt, unsigned G) {
  cbar();
  if (threadIdx.x == 0) {
    unsigned long long v, cur;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(v) : "l"(cnt) : "memory");
    const unsigned long long target = (v / G + 1) * G;
    do {
      asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(cnt) : "memory");
    } while (cur < target);
  }
  cbar();
}
}  // namespace

// Cross-warp flags in shared memory (producer / consumer hand-offs): every
// access after the CTA's initial barrier is an atomic, so the protocol is
// race-free in the memory model (and clean under compute-sanitizer racecheck).
__device__ __forceinline__ int flag_ld(volatile int* p) { return atomicAdd((int*)p, 0); }
__device__ __forceinline__ void flag_st(volatile int* p, int v) { atomicExch((int*)p, v); }
__device__ __forceinline__ long long flag_ld64(volatile long long* p) {
  return (long long)atomicAdd((unsigned long long*)p, 0ull);
}
__device__ __forceinline__ void flag_st64(volatile long long* p, long long v) {
  atomicExch((unsigned long long*)p, (unsigned long long)v);
}

__device__ __forceinline__ void tcg_final(const TcgState& s, int t, volatile int* sh_stop,
                                          TcgState* st) {
  if (t == 0) {
    flag_st(sh_stop, 1);
    if (blockIdx.x == 0) *st = s;
  }
}

struct TcgPersistArgs {
  const double* Q;
  int64_t ldq;
  int n, N;
  TcgState* st;
  const double* Y;
  const double* lam;
  double* res;                 // r_k (all rows; read by every CTA's stream)
  double* D0;                  // δ ping-pong: δ_k in D[k & 1]; D1 = 0 on entry (δ_{−1})
  double* D1;
  double* eta;
  double* Heta;
  double* QD;                  // Qδ rows (row producers → camera owners)
  double* pA;                  // per-CTA partials ⟨δ, Hδ⟩
  double* pB;                  // per-CTA partials ‖r‖²
  unsigned long long* gsync;   // grid barrier counter (0 on entry)
  unsigned long long* dbg;     // XM_PHASES: %globaltimer stamps [G][8] of iteration 1
  int bh;                      // rows per row block = the tensor map's box height
  int stages;                  // ring depth (full-row kernel; host-sized to the smem budget)
};

template <int R>
__global__ void __launch_bounds__(kPThreads, 1) k_tcg_persist(const __grid_constant__ CUtensorMap tmq,
                                                              TcgPersistArgs a) {
  // ring of S stages (runtime: as many as fit), stage = Q box (bh × 128) + r, δ chunks
  const int S = a.stages;
  const int stage_dbl = a.bh * kPCols + 2 * kPCols * R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stage_base = reinterpret_cast<double*>(smem_raw);
  uint64_t* fullQ = reinterpret_cast<uint64_t*>(stage_base + (size_t)S * stage_dbl);
  uint64_t* fullV = fullQ + S;
  uint64_t* empty = fullV + S;
  double* red = reinterpret_cast<double*>(empty + S);  // [2 halves][kBlockRows][R]
  double* acc = red + 2 * kBlockRows * R;              // [rows of this CTA][R]
  __shared__ TcgState ts;
  __shared__ volatile int sh_vgen;  // streams ≤ sh_vgen may load their r / δ tiles
  __shared__ volatile int sh_stop;
  __shared__ volatile long long sh_iq;      // Q copies issued for tiles < sh_iq
  __shared__ volatile long long sh_ivdone;  // V producer's final cursor (−1 while running)
  __shared__ double ws[kPW];

  const int G = gridDim.x;
  const int n = a.n;
  const int row_base = (int)((int64_t)blockIdx.x * n / G);
  const int nrow = (int)((int64_t)(blockIdx.x + 1) * n / G) - row_base;
  const int fa = (int)((int64_t)blockIdx.x * a.N / G);
  const int nf = (int)((int64_t)(blockIdx.x + 1) * a.N / G) - fa;
  const int bh = a.bh;                       // ≤ kBlockRows, same in every CTA
  const int nblocks = (nrow + bh - 1) / bh;
  const int nchunks = (n + kPCols - 1) / kPCols;
  const int tiles = nblocks * nchunks;  // per iteration
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&fullQ[s], 1);
      mbar_init(&fullV[s], 1);
      mbar_init(&empty[s], kPW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    ts = *a.st;
    sh_vgen = 0;
    sh_stop = ts.stop != 0;
    sh_iq = 0;
    sh_ivdone = -1;
  }
  __syncthreads();
  if (sh_stop) return;

  if (warp == kPW) {
    // ============================================================ Q producer
    // one 2-D tensor copy per stage: the row block (bh rows from the CTA's
    // block start; rows past the CTA's range are loaded and ignored, rows ≥ n
    // are zero-filled) × 128 columns
    if (lane != 0) return;
    const uint64_t pol_q = policy_evict_first();
    const unsigned qbytes = (unsigned)(kPCols * bh * 8);
    long long iq = 0;
    for (;; ++iq) {
      const int s = (int)(iq % S);
      const unsigned ph = (unsigned)((iq / S) & 1);
      bool go;
      while (!(go = mbar_try_wait(&empty[s], ph ^ 1u)))
        if (flag_ld(&sh_stop)) break;
      if (!go || flag_ld(&sh_stop)) break;
      const int tt = (int)(iq % tiles);
      const int b = tt / nchunks, j = tt % nchunks;
      mbar_expect_tx(&fullQ[s], qbytes);
      tma_load_2d(stage_base + (size_t)s * stage_dbl, &tmq, j * kPCols, row_base + b * bh,
                  &fullQ[s], pol_q);
      flag_st64(&sh_iq, iq + 1);
    }
    // Q copies issued for tiles nobody will consume must land first
    long long ivdone;
    while ((ivdone = flag_ld64(&sh_ivdone)) < 0) {
    }
    for (long long tq = ivdone; tq < iq; ++tq) mbar_wait(&fullQ[tq % S], (unsigned)((tq / S) & 1));
    return;
  }
  if (warp == kPW + 1) {
    // ======================================================= r / δ producer
    if (lane != 0) return;
    const uint64_t pol_v = policy_evict_last();
    long long iv = 0;
    int fenced = -1;
    for (;; ++iv) {
      const int kv = (int)(iv / tiles);
      bool stop = false;
      while (!(iv < flag_ld64(&sh_iq) && kv <= flag_ld(&sh_vgen))) {
        if (flag_ld(&sh_stop)) {
          stop = true;
          break;
        }
        __nanosleep(20);
      }
      if (stop) break;
      if (kv > fenced) {
        fence_proxy_async();  // r_k, δ_{k−1} were written by generic stores
        fenced = kv;
      }
      const int s = (int)(iv % S);
      const int j = (int)(iv % tiles) % nchunks;
      const int k0 = j * kPCols;
      const int klen = min(kPCols, n - k0);
      const unsigned vb = (unsigned)(((klen * R + 1) & ~1) * 8);
      double* st = stage_base + (size_t)s * stage_dbl + bh * kPCols;
      const double* dprev = (kv & 1) ? a.D0 : a.D1;  // δ_{k−1} = D[(k−1) & 1]
      mbar_expect_tx(&fullV[s], 2 * vb);
      tma_load_1d(st, a.res + (int64_t)k0 * R, vb, &fullV[s], pol_v);
      tma_load_1d(st + kPCols * R, dprev + (int64_t)k0 * R, vb, &fullV[s], pol_v);
    }
    flag_st64(&sh_ivdone, iv);  // tiles ≥ iv got no r / δ copy (and were never consumed)
    return;
  }

  // ================================================================== consumers
  // Camera state is (re)loaded after each stream — own rows of δ_k, r_k were
  // written by this same thread — so no registers are held across the stream.
  const int t = threadIdx.x;
  const bool has = t < nf;
  const int i = fa + t;
  if (has) {  // δ_0 = −r_0 (= fma(0, 0, −r): the same bits the streams form)
    Blk<R> r0b, d0b;
    load_blk<R>(a.res, i, r0b);
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) d0b.v[p][cc] = fma(0.0, 0.0, -r0b.v[p][cc]);
    store_blk<R>(a.D0, i, d0b);
  }
  double beta_prev = 0.0;  // β_{k−1}: stream k uses δ_k = −r_k + β_{k−1}δ_{k−1}
  const int quarter = warp >> 1, half = warp & 1;
  const int col = 64 * half + 2 * lane;  // this lane's column pair within a tile
  long long it = 0;
#define XM_PSTAMP(q) \
  if (a.dbg && k == 1 && t == 0) a.dbg[blockIdx.x * 8 + (q)] = gtimer();
  for (int k = 0;; ++k) {
    XM_PSTAMP(0);
    // ---------------------------------------------------------------- stream
    const double* dprev_g = (k & 1) ? a.D0 : a.D1;
    for (int b = 0; b < nblocks; ++b) {
      const int rb = min(bh, nrow - b * bh);       // valid rows of this block
      const int rq = (rb + 3) >> 2;                 // rows per quarter (≤ 12)
      const int q0 = quarter * rq;                  // this warp's first row in the block
      const int nq = max(0, min(rq, rb - q0));      // this warp's row count
      double acc12[kQuarterRows][R];
#pragma unroll
      for (int q = 0; q < kQuarterRows; ++q)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) acc12[q][cc] = 0.0;
      for (int j = 0; j < nchunks; ++j, ++it) {
        const int sidx = (int)(it % S);
        const unsigned ph = (unsigned)((it / S) & 1);
        mbar_wait(&fullQ[sidx], ph);
        mbar_wait(&fullV[sidx], ph);
        const int klen = min(kPCols, n - j * kPCols);
        const double* stg = stage_base + (size_t)sidx * stage_dbl;
        const double* rs = stg + bh * kPCols;
        const double* ds = rs + kPCols * R;
        const double* qrow = stg + (size_t)q0 * kPCols + col;
        if (col + 1 < klen) {
          double v0[R], v1[R];
#pragma unroll
          for (int cc = 0; cc < R; ++cc) {
            v0[cc] = fma(beta_prev, ds[col * R + cc], -rs[col * R + cc]);
            v1[cc] = fma(beta_prev, ds[(col + 1) * R + cc], -rs[(col + 1) * R + cc]);
          }
#pragma unroll
          for (int q = 0; q < kQuarterRows; ++q) {
            if (q < nq) {
              const double2 qv = *reinterpret_cast<const double2*>(qrow + q * kPCols);
#pragma unroll
              for (int cc = 0; cc < R; ++cc)
                acc12[q][cc] = fma(qv.x, v0[cc], fma(qv.y, v1[cc], acc12[q][cc]));
            }
          }
        } else if (col < klen) {
          double v0[R];
#pragma unroll
          for (int cc = 0; cc < R; ++cc) v0[cc] = fma(beta_prev, ds[col * R + cc], -rs[col * R + cc]);
#pragma unroll
          for (int q = 0; q < kQuarterRows; ++q) {
            if (q < nq) {
              const double qq = qrow[q * kPCols];
#pragma unroll
              for (int cc = 0; cc < R; ++cc) acc12[q][cc] = fma(qq, v0[cc], acc12[q][cc]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sidx]);
      }
      // reduce the row block: lanes (xor tree) → the two column halves (fixed order)
#pragma unroll
      for (int q = 0; q < kQuarterRows; ++q)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
          double v = acc12[q][cc];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          acc12[q][cc] = v;
        }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kQuarterRows; ++q)
          if (q < nq)
#pragma unroll
            for (int cc = 0; cc < R; ++cc) red[(half * kBlockRows + q0 + q) * R + cc] = acc12[q][cc];
      }
      cbar();
      for (int u = t; u < rb * R; u += kPC)
        acc[b * bh * R + u] = red[u] + red[kBlockRows * R + u];
      cbar();
    }
    XM_PSTAMP(1);
    // ------------------------------------------- rows → QD, ⟨δ_k, 2Qδ_k⟩ rows part
    double part = 0.0;
    for (int u = t; u < nrow * R; u += kPC) {
      const int64_t gidx = (int64_t)row_base * R + u;
      const double q = acc[u];
      a.QD[gidx] = q;
      const double d = fma(beta_prev, __ldcg(dprev_g + gidx), -__ldcg(a.res + gidx));  // δ_k
      part = fma(2.0 * q, d, part);
    }
    TcgState s = ts;
    Blk<R> y, dcur, rcur;
    double L[6];
    if (has) {  // camera part −2⟨δ_i, Λ_iδ_i⟩ (δ tangent, P self-adjoint)
      load_blk<R>(a.Y, i, y);
      load_blk<R>((k & 1) ? a.D1 : a.D0, i, dcur);  // δ_k = D[k & 1] (own rows)
      load_blk<R>(a.res, i, rcur);
#pragma unroll
      for (int q = 0; q < 6; ++q) L[q] = a.lam[6 * i + q];
      Blk<R> zero{}, lamd;
      sub_lam<R>(zero, L, dcur, 0.0, 1.0, lamd);
      part = fma(2.0, dotb<R>(dcur, lamd), part);
    }
    {
      const double pc = csum(part, ws);
      if (t == 0) a.pA[blockIdx.x] = pc;
    }
    XM_PSTAMP(2);
    cgrid_sync(a.gsync, G);
    XM_PSTAMP(3);
    // -------------------------------------------------- α, boundary / τ, update
    const double dHd = csum_partials(a.pA, G, ws);
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
    const double step = s.boundary ? s.tau : alpha;
    double rn2 = 0.0;
    if (has) {
      Blk<R> qv, hd, e, he;
      const double* qp = a.QD + (int64_t)3 * i * R;
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) qv.v[p][cc] = __ldcg(qp + p * R + cc);
      sub_lam<R>(qv, L, dcur, 2.0, 2.0, hd);  // Hδ = P(2Qδ − 2Λδ)
      project_blk<R>(y, i == 0, hd);
      load_blk<R>(a.eta, i, e);
      load_blk<R>(a.Heta, i, he);
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
          e.v[p][cc] = fma(step, dcur.v[p][cc], e.v[p][cc]);
          he.v[p][cc] = fma(step, hd.v[p][cc], he.v[p][cc]);
        }
      store_blk<R>(a.eta, i, e);
      store_blk<R>(a.Heta, i, he);
      if (!s.boundary) {
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int cc = 0; cc < R; ++cc) rcur.v[p][cc] = fma(step, hd.v[p][cc], rcur.v[p][cc]);
        project_blk<R>(y, i == 0, rcur);
        store_blk<R>(a.res, i, rcur);
        rn2 = frob2<R>(rcur);
      }
    }
    if (s.boundary) {
      tcg_final(s, t, &sh_stop, a.st);
      break;
    }
    {
      const double pr = csum(rn2, ws);
      if (t == 0) a.pB[blockIdx.x] = pr;
    }
    XM_PSTAMP(4);
    cgrid_sync(a.gsync, G);
    XM_PSTAMP(5);
    // ------------------------------------------------ stop tests, β, δ_{k+1}
    const double z = csum_partials(a.pB, G, ws);
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
    if (s.stop) {
      tcg_final(s, t, &sh_stop, a.st);
      break;
    }
    if (has) {
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) dcur.v[p][cc] = fma(s.beta, dcur.v[p][cc], -rcur.v[p][cc]);
      store_blk<R>((k & 1) ? a.D0 : a.D1, i, dcur);  // δ_{k+1} → D[(k+1) & 1]
    }
    beta_prev = s.beta;
    XM_PSTAMP(6);
    cbar();  // every consumer has read ts for this iteration
    if (t == 0) {
      ts = s;
      __threadfence_block();
      flag_st(&sh_vgen, k + 1);  // r_{k+1} and δ_k are final everywhere (barrier B)
    }
  }
  // (the break paths leave `s` in the loop scope: CTA 0 re-derives nothing —
  // it stored the final state before breaking, see tcg_final)
}

// ======================================================================
// Symmetric variant: the stream reads only the LOWER triangle of Q (half the
// bytes), with the tile geometry of the plain symmetric product (spmm_sym.cu):
// column panels J of 256 columns, each the run of 32-row tiles from its
// diagonal block down, numbered panel-major and split stream-K style into G
// equal contiguous ranges.  Per tile (warp w ↔ rows 4w … 4w+3, lane ℓ ↔
// columns {2ℓ+64m, 2ℓ+64m+1}): row part Σ_j Q_ij δ_j (butterfly reduce over
// the warp, one 32 × r partial per tile, row-tile-major), column part
// Σ_i Q_ij δ_i (registers over the CTA's run of the panel = a segment, one
// partial per segment).  δ_k is formed on the fly as fma(β, δ_{k−1}, −r_k) —
// for the panel's columns from L2 at segment start, for the tile's rows from
// the r / δ_{k−1} slices TMA-loaded next to the Q tile — with the fma the
// camera owners use, so every CTA sees bitwise the same δ (no third barrier).
// ⟨δ, Qδ⟩ = Σ δ_i·(row part) + Σ δ_j·(column part) comes out of the partials
// before barrier A; after it each CTA assembles the Qδ rows of its own
// cameras from the partials in a fixed order (deterministic).
//
// Thread 0 (of warp 0; no producer warp, so each thread may use 255
// registers) issues the copies: Q tiles run up to 3 stages ahead, across
// iterations (Q is constant); the r / δ slices of iteration k only after
// barrier B of k − 1 made r_k, δ_{k−1} final.
constexpr int kYR = 32;            // rows per tile (4 per warp)
constexpr int kYC = 256;           // panel width
constexpr int kYDiag = kYC / kYR;  // tiles of a panel's diagonal block
constexpr int kYS = 3;             // ring stages
constexpr int kYQDbl = kYR * kYC;  // Q tile (64 KB)
constexpr int kYStageDbl = kYQDbl + 2 * kYR * 5;  // + r, δ_{k−1} slices (r ≤ 5); 128-B multiple

struct SymTcgArgs {
  TcgPersistArgs b;
  const int* pbase;    // TCb + 1: first tile of panel J
  const int* tbase;    // G + 1: CTA c streams tiles [tbase[c], tbase[c+1]) (cost-balanced)
  const int* segbase;  // G + 1: first column-partial slot of CTA c
  const int* colptr;   // TCb + 1: slots [colptr[J], colptr[J+1]) hold panel J (consecutive)
  double* RP;          // [W][32][R] row partials, row-tile-major (rtile_base)
  double* CP;          // [slots][8 warps][R][256] column partials
  int TCb;
  int W;
  int pmax;            // assembly lanes per element, at most (1, 2, 4, …, 32)
};

// first row-part slot of row tile K: Σ_{K'<K} (⌊K'/8⌋ + 1)
__device__ __forceinline__ int64_t y_rtile_base(int K) {
  const int64_t a = K >> 3, b = K & 7;
  return (int64_t)K + 4 * a * (a - 1) + a * b;
}
__device__ __forceinline__ int y_panel_of(const int* __restrict__ pbase, int TCb, int t) {
  int lo = 0, hi = TCb - 1;  // largest J with pbase[J] ≤ t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(pbase + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// butterfly reduce-scatter of RP rows × R sums over the warp (spmm_sym.cu):
// lane ℓ ends with the sums of row ℓ >> (5 − log2 RP) in a[0][·]
template <int RP, int R>
__device__ __forceinline__ void y_rows_reduce(double (&a)[RP][R], int lane) {
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

template <int R>
__global__ void __launch_bounds__(kPC, 1) k_tcg_persist_sym(const __grid_constant__ CUtensorMap tmq,
                                                            SymTcgArgs sa) {
  constexpr int RP = (R <= 4) ? 4 : 2;  // rows reduced together (register budget)
  constexpr int S = kYS;
  const TcgPersistArgs& a = sa.b;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stage_base = reinterpret_cast<double*>(smem_raw);
  // one region, two uses: during the stream the next segment's column slices
  // (colv: r then δ_{k−1}, 256 × R each), after barrier A the Qδ rows of this
  // CTA's cameras (yown) — the stream never overlaps the camera phase
  double* colv = stage_base + (size_t)S * kYStageDbl;
  double* yown = colv;  // [3·cameras of this CTA][R]
  const int nf_max = (a.N + gridDim.x - 1) / gridDim.x;
  uint64_t* fullQ = reinterpret_cast<uint64_t*>(colv + max(3 * nf_max * R, 2 * kYC * R));
  uint64_t* fullV = fullQ + S;
  uint64_t* empty = fullV + S;
  uint64_t* colfull = empty + S;     // next segment's column slices landed
  uint64_t* colempty = colfull + 1;  // every warp has formed its δ_J registers from them
  __shared__ TcgState ts;
  __shared__ volatile int sh_stop;
  __shared__ double ws[kPW];

  const int G = gridDim.x;
  const int n = a.n;
  const int t0 = __ldg(sa.tbase + blockIdx.x);
  const int T = __ldg(sa.tbase + blockIdx.x + 1) - t0;  // tiles per iteration
  const int fa = (int)((int64_t)blockIdx.x * a.N / G);
  const int nf = (int)((int64_t)(blockIdx.x + 1) * a.N / G) - fa;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int J0 = (T > 0) ? y_panel_of(sa.pbase, sa.TCb, t0) : 0;

  if (t == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&fullQ[s], 1);
      mbar_init(&fullV[s], 1);
      mbar_init(&empty[s], kPW);
    }
    mbar_init(colfull, 1);
    mbar_init(colempty, kPW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    ts = *a.st;
    sh_stop = ts.stop != 0;
  }
  __syncthreads();
  if (sh_stop) return;
  // segments (panels J0 … J0 + nseg − 1) of this CTA's range, every iteration
  const int nseg = (T > 0) ? y_panel_of(sa.pbase, sa.TCb, t0 + T - 1) - J0 + 1 : 0;

  // ---------------------------------------------------------------- producer state (thread 0)
  // kept in shared memory: only thread 0 uses it, and registers are the
  // stream's budget (every thread is allocated what the busiest one needs)
  struct Prod {
    long long iq, iv;  // Q tiles / r,δ slices issued (global tile counter)
    long long ic;      // column-slice pairs issued (global segment counter)
    int qJ, qpend, vJ, vpend;
  };
  __shared__ Prod pr;
  // tile g of the CTA's cyclic sequence → (panel J, row tile); cursors walk
  // the panels incrementally and restart at J0 on every new iteration
  auto geo = [&](long long g, int& J, int& pend) {
    const int x = (int)(g % T);
    if (x == 0) {
      J = J0;
      pend = __ldg(sa.pbase + J0 + 1);
    }
    while (t0 + x >= pend) {
      ++J;
      pend = __ldg(sa.pbase + J + 1);
    }
    return kYDiag * J + (t0 + x - __ldg(sa.pbase + J));
  };
  auto issue_q = [&]() {
    const long long g = pr.iq;
    // the slot's previous tile (g − S) must be released by every consumer
    // warp (one completed phase of empty[s]; waited on every time, so no
    // phase of the barrier goes unobserved)
    if (g >= S) mbar_wait(&empty[g % S], (unsigned)(((g - S) / S) & 1));
    int J = pr.qJ, pend = pr.qpend;
    const int rt = geo(g, J, pend);
    pr.qJ = J;
    pr.qpend = pend;
    const int s = (int)(g % S);
    mbar_expect_tx(&fullQ[s], (unsigned)(kYQDbl * 8));
    tma_load_2d(stage_base + (size_t)s * kYStageDbl, &tmq, J * kYC, rt * kYR, &fullQ[s],
                policy_evict_first());
    pr.iq = g + 1;
  };
  auto issue_v = [&](int k) {
    const long long g = pr.iv;
    int J = pr.vJ, pend = pr.vpend;
    const int rt = geo(g, J, pend);
    pr.vJ = J;
    pr.vpend = pend;
    const int s = (int)(g % S);
    const int rlen = min(kYR, n - rt * kYR);
    const unsigned vb = (unsigned)(((rlen * R + 1) & ~1) * 8);
    const double* dprev = (k & 1) ? a.D0 : a.D1;  // δ_{k−1}
    double* st = stage_base + (size_t)s * kYStageDbl + kYQDbl;
    const uint64_t pol_v = policy_evict_last();
    mbar_expect_tx(&fullV[s], 2 * vb);
    tma_load_1d(st, a.res + (int64_t)rt * kYR * R, vb, &fullV[s], pol_v);
    tma_load_1d(st + kYR * R, dprev + (int64_t)rt * kYR * R, vb, &fullV[s], pol_v);
    pr.iv = g + 1;
  };
  // next segment's column slices, once the previous ones were consumed and
  // the segment belongs to iteration k (its r_k, δ_{k−1} are final)
  auto issue_col = [&](int k) {
    const long long g = pr.ic;
    if (g >= (long long)(k + 1) * nseg) return;
    if (g > 0 && !mbar_test(colempty, (unsigned)((g - 1) & 1))) return;
    const int J = J0 + (int)(g % nseg);
    const int nj = min(kYC, n - J * kYC);
    const unsigned cb = (unsigned)(((nj * R + 1) & ~1) * 8);
    const double* dprev = (k & 1) ? a.D0 : a.D1;
    const uint64_t pol_v = policy_evict_last();
    mbar_expect_tx(colfull, 2 * cb);
    tma_load_1d(colv, a.res + (int64_t)J * kYC * R, cb, colfull, pol_v);
    tma_load_1d(colv + kYC * R, dprev + (int64_t)J * kYC * R, cb, colfull, pol_v);
    pr.ic = g + 1;
  };
  if (t == 0) {
    pr.iq = 0;
    pr.iv = 0;
    pr.ic = 0;
    pr.qJ = pr.vJ = J0;
    pr.qpend = pr.vpend = 0;
    if (T > 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmq)) : "memory");
      for (int q = 0; q < S; ++q) issue_q();
    }
  }

  // ---------------------------------------------------------------- camera owners
  const bool has = t < nf;
  const int i = fa + t;
  if (has) {  // δ_0 = −r_0
    Blk<R> r0b, d0b;
    load_blk<R>(a.res, i, r0b);
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) d0b.v[p][cc] = fma(0.0, 0.0, -r0b.v[p][cc]);
    store_blk<R>(a.D0, i, d0b);
  }
  double beta_prev = 0.0;
  long long it = 0;  // tiles consumed (global)
  for (int k = 0;; ++k) {
    XM_PSTAMP(0);
    if (t == 0 && T > 0) {  // this iteration's r / δ_{k−1} slices (after barrier B of k − 1)
      fence_proxy_async();
      issue_col(k);
      while (pr.iv < pr.iq && pr.iv < (long long)(k + 1) * T) issue_v(k);
    }
    // ------------------------------------------------------------ stream Qδ_k
    double part = 0.0;  // this thread's share of ⟨δ_k, Qδ_k⟩
    double vr[8][R], colacc[8][R];
    int J = -1, pend = 0, seg = 0;
    auto flush = [&]() {
      // ⟨δ_J, column part⟩ per lane; each warp writes its own column partial
      // (no cross-warp step here: the assembly sums the 8 warps in order)
#pragma unroll
      for (int m = 0; m < 8; ++m)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) part = fma(vr[m][cc], colacc[m][cc], part);
      // layout [slot][warp][cc][col]: a lane's column pair is one 16-B store
      double* dst = sa.CP + ((int64_t)(__ldg(sa.segbase + blockIdx.x) + seg - 1) * kPW + warp) * R * kYC;
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int cc = 0; cc < R; ++cc)
          *reinterpret_cast<double2*>(dst + cc * kYC + 2 * lane + 64 * m) =
              make_double2(colacc[2 * m][cc], colacc[2 * m + 1][cc]);
    };
    auto do_rows = [&](auto diag_tag, const double* st, const double* rI, const double* dI, int nv,
                       int k0, int dl0, double* rp) {
      constexpr bool DIAG = decltype(diag_tag)::value;
      double rs[RP][R];
#pragma unroll
      for (int kk = 0; kk < RP; ++kk) {
        const int rl = 4 * warp + k0 + kk;
        const double* q = st + rl * kYC;
        double vrow[R];
#pragma unroll
        for (int cc = 0; cc < R; ++cc)
          vrow[cc] = (rl < nv) ? fma(beta_prev, dI[rl * R + cc], -rI[rl * R + cc]) : 0.0;
        const int dl = dl0 + rl;
#pragma unroll
        for (int cc = 0; cc < R; ++cc) rs[kk][cc] = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int jl = 2 * lane + 64 * m;
          const double2 q2 = *reinterpret_cast<const double2*>(q + jl);
          double qa = q2.x, qb = q2.y, ca = qa, cb = qb;
          if (DIAG) {  // row part j ≤ i, column part j < i
            qa = (jl <= dl) ? qa : 0.0;
            qb = (jl + 1 <= dl) ? qb : 0.0;
            ca = (jl < dl) ? q2.x : 0.0;
            cb = (jl + 1 < dl) ? q2.y : 0.0;
          }
#pragma unroll
          for (int cc = 0; cc < R; ++cc) {
            rs[kk][cc] = fma(qa, vr[2 * m][cc], fma(qb, vr[2 * m + 1][cc], rs[kk][cc]));
            colacc[2 * m][cc] = fma(ca, vrow[cc], colacc[2 * m][cc]);
            colacc[2 * m + 1][cc] = fma(cb, vrow[cc], colacc[2 * m + 1][cc]);
          }
        }
      }
      y_rows_reduce<RP, R>(rs, lane);
      constexpr int sh = (RP == 4) ? 3 : (RP == 2 ? 4 : 5);
      if ((lane & ((1 << sh) - 1)) == 0) {
        const int rl = 4 * warp + k0 + (lane >> sh);
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
          rp[rl * R + cc] = rs[0][cc];
          const double di = (rl < nv) ? fma(beta_prev, dI[rl * R + cc], -rI[rl * R + cc]) : 0.0;
          part = fma(di, rs[0][cc], part);
        }
      }
    };
    for (int x = 0; x < T; ++x, ++it) {
      const int tt = t0 + x;
      if (tt >= pend) {  // new segment: flush the previous one, form δ_J for the lane's columns
        if (J >= 0) flush();
        J = (J < 0) ? J0 : J + 1;
        pend = __ldg(sa.pbase + J + 1);
        const int nj = min(kYC, n - J * kYC);
        const long long gs = (long long)k * nseg + seg;  // global segment index
        mbar_wait(colfull, (unsigned)(gs & 1));
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jl = 2 * lane + 64 * m + h;
#pragma unroll
            for (int cc = 0; cc < R; ++cc) {
              vr[2 * m + h][cc] =
                  (jl < nj) ? fma(beta_prev, colv[kYC * R + jl * R + cc], -colv[jl * R + cc]) : 0.0;
              colacc[2 * m + h][cc] = 0.0;
            }
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(colempty);
        ++seg;
      }
      const int ptl = tt - __ldg(sa.pbase + J);  // tile within the panel
      const int rt = kYDiag * J + ptl;
      const int s = (int)(it % S);
      const unsigned ph = (unsigned)((it / S) & 1);
      mbar_wait(&fullQ[s], ph);
      mbar_wait(&fullV[s], ph);
      const double* st = stage_base + (size_t)s * kYStageDbl;
      const double* rI = st + kYQDbl;
      const double* dI = rI + kYR * R;
      const int nv = n - rt * kYR;
      double* rp = sa.RP + (y_rtile_base(rt) + J) * kYR * R;
      if (ptl < kYDiag) {
#pragma unroll
        for (int k0 = 0; k0 < 4; k0 += RP) do_rows(std::true_type{}, st, rI, dI, nv, k0, ptl * kYR, rp);
      } else {
#pragma unroll
        for (int k0 = 0; k0 < 4; k0 += RP) do_rows(std::false_type{}, st, rI, dI, nv, k0, 0, rp);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (t == 0) {
        // refill slot s with the tile S ahead if it belongs to this iteration;
        // the next iteration's first tiles are issued after the assembly
        // (in flight during barriers they would queue ahead of its L2 reads)
        if (it + S < (long long)(k + 1) * T) {
          issue_q();  // waits for empty[s] (phase ph) itself
          if (pr.iv < pr.iq) issue_v(k);
        }
        if (pr.ic < (long long)(k + 1) * nseg) issue_col(k);
      }
    }
    if (J >= 0) flush();
    XM_PSTAMP(1);
    TcgState s = ts;
    Blk<R> y, dcur, rcur;
    double L[6];
    if (has) {
      load_blk<R>(a.Y, i, y);
      load_blk<R>((k & 1) ? a.D1 : a.D0, i, dcur);
      load_blk<R>(a.res, i, rcur);
#pragma unroll
      for (int q = 0; q < 6; ++q) L[q] = a.lam[6 * i + q];
    }
    {  // ⟨δ, Hδ⟩ = 2⟨δ, Qδ⟩ − 2⟨δ, Λδ⟩ (δ tangent, P orthogonal)
      double cam = 0.0;
      if (has) {
        Blk<R> zero{}, lamd;
        sub_lam<R>(zero, L, dcur, 0.0, 1.0, lamd);
        cam = dotb<R>(dcur, lamd);
      }
      const double pc = csum(fma(2.0, part, 2.0 * cam), ws);
      if (t == 0) a.pA[blockIdx.x] = pc;
    }
    XM_PSTAMP(2);
    cgrid_sync(a.gsync, G);
    XM_PSTAMP(3);
    // ---------------------- assemble Qδ at this CTA's camera rows (fixed order)
    // every load of an element in flight at once (latency, not bandwidth,
    // bounds this phase); this thread's ⟨δ,Hδ⟩ partial load overlaps it
    const double pa_mine = (t < G) ? __ldcg(a.pA + t) : 0.0;  // = csum_partials' assignment (G ≤ 256)
    // P consecutive lanes per element (P·elements ≤ 256, P ≤ sa.pmax): lane
    // j of a group sums list items j, j+P, … (batches of 32 loads in flight),
    // then a fixed xor tree over the group.  The loop trip count is
    // warp-uniform (the shuffles need every lane).
    const int ne = 3 * nf * R;
    int P = 1;
    while (P < sa.pmax && 2 * P * ne <= kPC) P *= 2;
    for (int ob = (t >> 5) * (32 / P); ob < ne; ob += kPC / P) {
      const int o = ob + lane / P, j = lane % P;
      const bool ok = o < ne;
      const int oo = ok ? o : 0;
      const int row = 3 * fa + oo / R, cc = oo % R;
      const int K = row / kYR, l = row % kYR, Jc = row / kYC, mcol = row % kYC;
      const double* p = sa.RP + (y_rtile_base(K) * kYR + l) * R + cc;
      constexpr int64_t st = kYR * R;
      const int nrp = ok ? Jc + 1 : 0;
      double y2 = 0.0;
      for (int q0 = j; q0 < nrp; q0 += 32 * P) {  // panels (zeros past Jc add exactly)
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = (q0 + u * P < nrp) ? __ldcg(p + (int64_t)(q0 + u * P) * st) : 0.0;
#pragma unroll
        for (int u = 0; u < 32; ++u) y2 += v[u];
      }
      // column partials of panel Jc: (slot, warp) pairs in order — consecutive
      // in the [slot][warp][cc][col] layout
      const int f0 = __ldg(sa.colptr + Jc) * kPW, nfl = ok ? __ldg(sa.colptr + Jc + 1) * kPW - f0 : 0;
      const double* c = sa.CP + ((int64_t)f0 * R + cc) * kYC + mcol;
      for (int q0 = j; q0 < nfl; q0 += 32 * P) {
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u)
          v[u] = (q0 + u * P < nfl) ? __ldcg(c + (int64_t)(q0 + u * P) * R * kYC) : 0.0;
#pragma unroll
        for (int u = 0; u < 32; ++u) y2 += v[u];
      }
      for (int o2 = 1; o2 < P; o2 <<= 1) y2 += __shfl_xor_sync(0xffffffffu, y2, o2);
      if (ok && j == 0) yown[o] = y2;
    }
    // -------------------------------------------------- α, boundary / τ, update
    const double dHd = csum(pa_mine, ws);  // its cbar also publishes yown
    XM_PSTAMP(7);
    if (t == 0 && T > 0)  // Q prefetch of the next iteration (every warp has released every slot)
      while (pr.iq < it + S) issue_q();
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
    const double step = s.boundary ? s.tau : alpha;
    double rn2 = 0.0;
    if (has) {
      Blk<R> qv, hd, e, he;
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) qv.v[p][cc] = yown[(3 * t + p) * R + cc];
      sub_lam<R>(qv, L, dcur, 2.0, 2.0, hd);  // Hδ = P(2Qδ − 2Λδ)
      project_blk<R>(y, i == 0, hd);
      load_blk<R>(a.eta, i, e);
      load_blk<R>(a.Heta, i, he);
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
          e.v[p][cc] = fma(step, dcur.v[p][cc], e.v[p][cc]);
          he.v[p][cc] = fma(step, hd.v[p][cc], he.v[p][cc]);
        }
      store_blk<R>(a.eta, i, e);
      store_blk<R>(a.Heta, i, he);
      if (!s.boundary) {
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int cc = 0; cc < R; ++cc) rcur.v[p][cc] = fma(step, hd.v[p][cc], rcur.v[p][cc]);
        project_blk<R>(y, i == 0, rcur);
        store_blk<R>(a.res, i, rcur);
        rn2 = frob2<R>(rcur);
      }
    }
    if (s.boundary) {
      tcg_final(s, t, &sh_stop, a.st);
      break;
    }
    {
      const double pr = csum(rn2, ws);
      if (t == 0) a.pB[blockIdx.x] = pr;
    }
    XM_PSTAMP(4);
    cgrid_sync(a.gsync, G);
    XM_PSTAMP(5);
    const double z = csum_partials(a.pB, G, ws);
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
    if (s.stop) {
      tcg_final(s, t, &sh_stop, a.st);
      break;
    }
    if (has) {
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int cc = 0; cc < R; ++cc) dcur.v[p][cc] = fma(s.beta, dcur.v[p][cc], -rcur.v[p][cc]);
      store_blk<R>((k & 1) ? a.D0 : a.D1, i, dcur);  // δ_{k+1} → D[(k+1) & 1]
    }
    beta_prev = s.beta;
    XM_PSTAMP(6);
    cbar();
    if (t == 0) ts = s;
    cbar();
  }
  // drain: no Q copy may still be landing in shared memory when the CTA exits
  if (t == 0)
    for (long long g = it; g < pr.iq; ++g) mbar_wait(&fullQ[g % S], (unsigned)((g / S) & 1));
}

// ---------------------------------------------------------------------- host
namespace {
constexpr size_t kSmemCap = 227 * 1024 - 1024;  // dynamic budget (static smem ≈ 0.3 KB)
int persist_bh_(int n, int G) {
  const int rows_max = ceil_div(n, G);
  return ceil_div(rows_max, ceil_div(rows_max, kBlockRows));
}
// ring depth: as many stages (≤ 6) as fit next to the reduction scratch
template <int R>
int persist_stages(int n, int G) {
  const size_t stage = (size_t)8 * (persist_bh_(n, G) * kPCols + 2 * kPCols * R);
  const size_t other = (size_t)2 * kBlockRows * R * 8 + (size_t)(ceil_div(n, G) + 1) * R * 8;
  const long long s = ((long long)kSmemCap - (long long)other) / (long long)(stage + 24);
  static const long long cap = [] {  // XM_PERSIST_STAGES: A/B switch for measurements
    const char* e = std::getenv("XM_PERSIST_STAGES");
    return e ? std::max(2ll, std::atoll(e)) : 4ll;
  }();
  return (int)std::max(0ll, std::min(cap, s));
}
template <int R>
size_t persist_smem(int n, int G) {
  const int S = persist_stages<R>(n, G);
  if (S < 2) return ~(size_t)0;
  const size_t stage = (size_t)8 * (persist_bh_(n, G) * kPCols + 2 * kPCols * R);
  return (size_t)S * stage + 3 * (size_t)S * 8 + (size_t)2 * kBlockRows * R * 8 +
         (size_t)(ceil_div(n, G) + 1) * R * 8;
}
size_t persist_smem_r(int r, int n, int G) {
  switch (r) {
    case 1: return persist_smem<1>(n, G);
    case 2: return persist_smem<2>(n, G);
    case 3: return persist_smem<3>(n, G);
    case 4: return persist_smem<4>(n, G);
    case 5: return persist_smem<5>(n, G);
    default: return ~(size_t)0;
  }
}
}  // namespace

bool tcg_persist_sym_supported(xm_ctx* c, int r);

bool tcg_persist_supported(xm_ctx* c, int r) {
  if (tcg_persist_sym_supported(c, r)) return true;
  if (!c->fused_tcg || !c->persist_tcg || c->world != 1 || r < 1 || r > 5 ||
      !tcg_fullrow_ok(c) || c->N < 1 || !fused_epilogues(c))
    return false;
  const int G = std::min(148, c->N);
  return ceil_div(c->N, G) <= kPC && persist_smem_r(r, c->n, G) <= kSmemCap;
}

// rows per block: the CTA row count (⌈n/G⌉) split into ⌈·/48⌉ equal blocks
static int persist_bh(int n, int G) {
  const int rows_max = ceil_div(n, G);
  return ceil_div(rows_max, ceil_div(rows_max, kBlockRows));
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
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
  return encode;
}

// Q as a 2-D tensor (n columns × n rows, row pitch ldq·8), box kPCols × bh,
// rows / columns ≥ n zero-filled.  Cached in `raw` (128 B) per (Q, bh, n).
static const CUtensorMap* q_tmap(xm_ctx* c, int bh, unsigned char* raw, const void** q_cached,
                                 int* bh_cached, int* n_cached) {
  if (*q_cached == c->Q.p && *bh_cached == bh && *n_cached == c->n)
    return reinterpret_cast<const CUtensorMap*>(raw);
  cuuint64_t dims[2] = {(cuuint64_t)c->n, (cuuint64_t)c->n};
  cuuint64_t strides[1] = {(cuuint64_t)c->ldq * 8};
  cuuint32_t box[2] = {(cuuint32_t)kPCols, (cuuint32_t)bh};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tmap_encoder()(reinterpret_cast<CUtensorMap*>(raw), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                              c->Q.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(XM_ECUDA, "cuTensorMapEncodeTiled failed (persistent tCG)");
  *q_cached = c->Q.p;
  *bh_cached = bh;
  *n_cached = c->n;
  return reinterpret_cast<const CUtensorMap*>(raw);
}

static const CUtensorMap* persist_tmap(xm_ctx* c, int G) {
  return q_tmap(c, persist_bh(c->n, G), c->persist_tmap, &c->persist_tmap_q, &c->persist_tmap_bh,
                &c->persist_tmap_n);
}

template <int R>
static void launch_persist(xm_ctx* c) {
  const int G = std::min(148, c->N);
  const CUtensorMap* tm = persist_tmap(c, G);
  const size_t smem = persist_smem<R>(c->n, G);
  if (smem > kSmemCap) throw Error(XM_EINVAL, "persistent tCG shared memory plan exceeds 227 KB");
  ensure_smem_attr((const void*)k_tcg_persist<R>, smem);
  TcgPersistArgs a{};
  a.Q = c->Q.p;
  a.ldq = c->ldq;
  a.n = c->n;
  a.N = c->N;
  a.st = c->tcg.p;
  a.Y = c->Y.p;
  a.lam = c->lam.p;
  a.res = c->res.p;
  a.D0 = c->dir.p;
  a.D1 = c->dir2.p;
  a.eta = c->eta.p;
  a.Heta = c->Heta.p;
  a.QD = c->Hdir.p;
  a.pA = c->part1.p;
  a.pB = c->part2.p;
  a.gsync = c->gsync.p;
  a.bh = c->persist_tmap_bh;
  a.stages = persist_stages<R>(c->n, G);
  if (c->phases_on) {
    if (!c->tdbg.p) {
      c->tdbg.alloc(148 * 8);
      XM_CUDA(cudaMemsetAsync(c->tdbg.p, 0, 148 * 8 * 8, c->stream));
    }
    a.dbg = c->tdbg.p;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  XM_CUDA(cudaLaunchKernelEx(&cfg, k_tcg_persist<R>, *tm, a));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

// Whole tCG solve (state already initialised by tcg_init); returns after the
// kernel is enqueued.  Algorithmic bytes per iteration for the roofline:
// Q (8·n·n) + the r and δ tiles every CTA streams (2·8·n·r per CTA row group,
// from L2) are not HBM-unique; we count Q + one pass over r, δ, QD, η, Hη, Y
// (8·n·r each, ≈ 9·8·n·r with reads + writes) + Λ (48·N).
double tcg_persist_bytes_per_iter(xm_ctx* c, int r) {
  const double n = c->n;
  const double qb = tcg_persist_sym_supported(c, r) ? 8.0 * n * (n + 1) / 2 : 8.0 * n * n;
  return qb + 9.0 * 8.0 * n * r + 48.0 * c->N;
}

// ------------------------------------------------------------- symmetric host
// Work plan of k_tcg_persist_sym for (n, G): panel bases, per-CTA column-partial
// slot bases, the slots of each panel, the 256 × 32 Q tensor map, partials.
struct SymTcgPlan {
  int n = 0, G = 0, TCb = 0, W = 0, slots = 0;
  DBuf<int> pbase, tbase, segbase, colptr;
  DBuf<double> RP, CP;
  alignas(64) unsigned char tmap[128] = {0};
  const void* tmap_q = nullptr;
  int64_t tmap_ld = 0;
};

static SymTcgPlan& sym_tcg_plan(xm_ctx* c) {
  if (!c->persist_sym_plan) c->persist_sym_plan = new SymTcgPlan();
  SymTcgPlan& p = *static_cast<SymTcgPlan*>(c->persist_sym_plan);
  const int n = c->n, G = std::min(148, c->N);
  if (p.n != n || p.G != G) {
    p.n = n;
    p.G = G;
    const int TRt = ceil_div(n, kYR);
    p.TCb = ceil_div(n, kYC);
    std::vector<int> pb(p.TCb + 1, 0);
    for (int J = 0; J < p.TCb; ++J) pb[J + 1] = pb[J] + (TRt - kYDiag * J);
    p.W = pb[p.TCb];
    // cost-balanced split: a tile costs 1, a diagonal-block tile 1 + c_d
    // (masks), the first tile of a panel 1 + c_s (a CTA crossing into a new
    // panel flushes a column partial and starts a segment); measured at B
    // with XM_PHASES_CTA: a second segment ≈ +1.5 tiles of stream time
    double cs = 1.5, cd = 0.1;
    if (const char* e = std::getenv("XM_PSYM_CSEG")) cs = atof(e);
    if (const char* e = std::getenv("XM_PSYM_CDIAG")) cd = atof(e);
    std::vector<double> cum(p.W + 1, 0.0);
    for (int J = 0, tt = 0; J < p.TCb; ++J)
      for (int x = 0; x < pb[J + 1] - pb[J]; ++x, ++tt)
        cum[tt + 1] = cum[tt] + 1.0 + (x < kYDiag ? cd : 0.0) + (x == 0 ? cs : 0.0);
    std::vector<int> tb(G + 1, 0);
    for (int cta = 1; cta < G; ++cta) {
      const double target = cum[p.W] * cta / G;
      int tt = tb[cta - 1];
      while (tt < p.W && cum[tt] < target) ++tt;
      tb[cta] = tt;
    }
    tb[G] = p.W;
    std::vector<int> sb(G + 1, 0), segpanel;
    for (int cta = 0; cta < G; ++cta) {
      const int64_t t0 = tb[cta], t1 = tb[cta + 1];
      sb[cta] = (int)segpanel.size();
      int J = 0;
      for (int64_t tt = t0; tt < t1;) {
        while (pb[J + 1] <= tt) ++J;
        segpanel.push_back(J);
        tt = std::min<int64_t>(t1, pb[J + 1]);
      }
    }
    sb[G] = (int)segpanel.size();
    p.slots = sb[G];
    std::vector<int> cp(p.TCb + 1, 0);
    for (int s = 0, J = 0; J <= p.TCb; ++J) {  // segpanel is non-decreasing
      while (s < p.slots && segpanel[s] < J) ++s;
      cp[J] = s;
    }
    p.pbase.alloc(pb.size());
    p.tbase.alloc(tb.size());
    XM_CUDA(cudaMemcpy(p.tbase.p, tb.data(), tb.size() * 4, cudaMemcpyHostToDevice));
    p.segbase.alloc(sb.size());
    p.colptr.alloc(cp.size());
    XM_CUDA(cudaMemcpy(p.pbase.p, pb.data(), pb.size() * 4, cudaMemcpyHostToDevice));
    XM_CUDA(cudaMemcpy(p.segbase.p, sb.data(), sb.size() * 4, cudaMemcpyHostToDevice));
    XM_CUDA(cudaMemcpy(p.colptr.p, cp.data(), cp.size() * 4, cudaMemcpyHostToDevice));
  }
  p.RP.alloc((size_t)p.W * kYR * 5 + 64);  // sized for r ≤ 5 (fixed addresses)
  p.CP.alloc((size_t)std::max(p.slots, 1) * kPW * kYC * 5 + 64);
  if (p.tmap_q != c->Q.p || p.tmap_ld != c->ldq) {  // box 256 × 32, rows / columns ≥ n zero-filled
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)c->ldq * 8};
    cuuint32_t box[2] = {(cuuint32_t)kYC, (cuuint32_t)kYR};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = tmap_encoder()(reinterpret_cast<CUtensorMap*>(p.tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                                c->Q.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(XM_ECUDA, "cuTensorMapEncodeTiled failed (symmetric tCG)");
    p.tmap_q = c->Q.p;
    p.tmap_ld = c->ldq;
  }
  return p;
}

void sym_tcg_plan_destroy(xm_ctx* c) {
  delete static_cast<SymTcgPlan*>(c->persist_sym_plan);
  c->persist_sym_plan = nullptr;
}

namespace {
template <int R>
size_t persist_sym_smem(int N, int G) {
  const int nf_max = ceil_div(N, G);
  return (size_t)kYS * kYStageDbl * 8 + std::max((size_t)3 * nf_max * R * 8, (size_t)2 * kYC * R * 8) +
         (3 * kYS + 2) * 8;
}
size_t persist_sym_smem_r(int r, int N, int G) {
  switch (r) {
    case 1: return persist_sym_smem<1>(N, G);
    case 2: return persist_sym_smem<2>(N, G);
    case 3: return persist_sym_smem<3>(N, G);
    case 4: return persist_sym_smem<4>(N, G);
    case 5: return persist_sym_smem<5>(N, G);
    default: return ~(size_t)0;
  }
}
}  // namespace

// Default below N = 4000 (B: 46.8 vs 53.0 µs per tCG iteration for the
// full-row kernel, same box); at E the three-kernel iteration around the
// plain symmetric product wins (605 vs 708 µs: 69 cameras per CTA to
// assemble, spills at r = 4).
bool tcg_persist_sym_supported(xm_ctx* c, int r) {
  if (c->persist_sym < 0 || !c->fused_tcg || !c->persist_tcg || c->world != 1 || r < 1 || r > 5 ||
      c->N < 1 || c->opt.spmm_kernel == 1 || !fused_epilogues(c))
    return false;
  if (c->persist_sym == 0 && c->N >= 4000) return false;
  const int G = std::min(148, c->N);
  return ceil_div(c->N, G) <= kPC && persist_sym_smem_r(r, c->N, G) <= kSmemCap;
}

template <int R>
static void launch_persist_sym(xm_ctx* c) {
  const int G = std::min(148, c->N);
  SymTcgPlan& p = sym_tcg_plan(c);
  const size_t smem = persist_sym_smem<R>(c->N, G);
  if (smem > kSmemCap) throw Error(XM_EINVAL, "symmetric persistent tCG smem plan exceeds 227 KB");
  ensure_smem_attr((const void*)k_tcg_persist_sym<R>, smem);
  SymTcgArgs sa{};
  TcgPersistArgs& a = sa.b;
  a.Q = c->Q.p;
  a.ldq = c->ldq;
  a.n = c->n;
  a.N = c->N;
  a.st = c->tcg.p;
  a.Y = c->Y.p;
  a.lam = c->lam.p;
  a.res = c->res.p;
  a.D0 = c->dir.p;
  a.D1 = c->dir2.p;
  a.eta = c->eta.p;
  a.Heta = c->Heta.p;
  a.QD = c->Hdir.p;
  a.pA = c->part1.p;
  a.pB = c->part2.p;
  a.gsync = c->gsync.p;
  a.bh = kYR;
  if (c->phases_on) {
    if (!c->tdbg.p) {
      c->tdbg.alloc(148 * 8);
      XM_CUDA(cudaMemsetAsync(c->tdbg.p, 0, 148 * 8 * 8, c->stream));
    }
    a.dbg = c->tdbg.p;
  }
  sa.pbase = p.pbase.p;
  sa.tbase = p.tbase.p;
  sa.segbase = p.segbase.p;
  sa.colptr = p.colptr.p;
  sa.RP = p.RP.p;
  sa.CP = p.CP.p;
  sa.TCb = p.TCb;
  sa.W = p.W;
  sa.pmax = 32;
  if (const char* e = std::getenv("XM_PSYM_PMAX")) sa.pmax = std::max(1, std::min(32, atoi(e)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kPC);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  XM_CUDA(cudaLaunchKernelEx(&cfg, k_tcg_persist_sym<R>, *reinterpret_cast<const CUtensorMap*>(p.tmap), sa));
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void tcg_persist_launch(xm_ctx* c, int r) {
  if (tcg_persist_sym_supported(c, r)) {
    const int64_t len = (int64_t)c->n * r;
    c->dir2.alloc((size_t)len + 64);
    XM_CUDA(cudaMemsetAsync(c->dir2.p, 0, len * 8, c->stream));  // δ_{−1} = 0
    switch (r) {
      case 1: launch_persist_sym<1>(c); return;
      case 2: launch_persist_sym<2>(c); return;
      case 3: launch_persist_sym<3>(c); return;
      case 4: launch_persist_sym<4>(c); return;
      case 5: launch_persist_sym<5>(c); return;
    }
  }
  const int64_t len = (int64_t)c->n * r;
  c->dir2.alloc((size_t)len + 64);
  XM_CUDA(cudaMemsetAsync(c->dir2.p, 0, len * 8, c->stream));  // δ_{−1} = 0
  switch (r) {
    case 1: launch_persist<1>(c); break;
    case 2: launch_persist<2>(c); break;
    case 3: launch_persist<3>(c); break;
    case 4: launch_persist<4>(c); break;
    case 5: launch_persist<5>(c); break;
    default: throw Error(XM_EINVAL, "persistent tCG supports r ≤ 5");
  }
}

}  // namespace xm
