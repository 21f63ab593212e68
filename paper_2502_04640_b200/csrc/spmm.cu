// spmm.cu — H6: out = Q·V for the tall-skinny BM factor V ∈ ℝ^{n×r}
// (cost, gradient, every HVP of tCG, Δf, escapes, Lanczos with r = 1).
// The paper applies its dense Q with cuBLAS matrix-vector products (P:520,
// P:1075); here one streaming kernel reads each Q byte exactly once per product.
//
// Roofline: HBM-bound.  Algorithmic bytes per product = 8·nrows·n (Q) +
// 8·n·r (V) + 8·nrows·r (out); 2·nrows·n·r flop ⇒ 0.25·r flop/B, far below the
// fp64 ridge (≈6 flop/B), so tensor cores are irrelevant.
//
// Design (sm_100a):
//  * grid = (row blocks) × (K splits); a CTA streams its row range of one K
//    chunk.  The V chunk (kc × r) is staged once per CTA in shared memory,
//    transposed (Vt[c][k]) so that every lane reads a conflict-free double2.
//  * each warp owns a contiguous slice of the CTA's rows and processes RPW rows
//    at a time: per 64-column step a lane issues RPW 128-bit streaming loads
//    (ld.global.cs: evict-first, Q must not evict V / partials from L2) and
//    r shared-memory double2 loads, 2·RPW·r FMAs.
//  * per row group the lane partials are reduced with warp shuffles.
//  * split-K partials are summed in a fixed order by spmm_reduce (deterministic;
//    identical row results for any number of ranks).
//  * grid sized to whole waves of 148 SMs × resident CTAs.
#include "xm_internal.cuh"

namespace xm {

constexpr int kSpmmThreads = 256;
constexpr int kSpmmWarps = kSpmmThreads / 32;

template <int R, int RPW>
__global__ void __launch_bounds__(kSpmmThreads) k_spmm_partial(
    const double* __restrict__ Q, int64_t ldq, int nrows, int n, const double* __restrict__ V,
    int kc, int nrowblk, double* __restrict__ part, const int* __restrict__ stop,
    int* __restrict__ exec_flag) {
  if (stop && *stop) return;
  if (exec_flag && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *exec_flag = 1;
  extern __shared__ __align__(16) double vt[];  // [R][kc]
  const int rb = blockIdx.x, split = blockIdx.y;
  const int k0 = split * kc;
  const int klen = min(kc, n - k0);
  // stage V chunk transposed
  for (int idx = threadIdx.x; idx < klen * R; idx += kSpmmThreads) {
    int k = idx / R, cc = idx - k * R;
    vt[cc * kc + k] = V[(int64_t)(k0 + k) * R + cc];
  }
  __syncthreads();
  const int r_lo = (int)((int64_t)rb * nrows / nrowblk);
  const int r_hi = (int)((int64_t)(rb + 1) * nrows / nrowblk);
  const int cnt = r_hi - r_lo;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w_lo = r_lo + (int)((int64_t)warp * cnt / kSpmmWarps);
  const int w_hi = r_lo + (int)((int64_t)(warp + 1) * cnt / kSpmmWarps);
  const int kfull = klen & ~63;  // columns covered by full 64-wide steps
  for (int row = w_lo; row < w_hi; row += RPW) {
    double acc[RPW][R];
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) acc[q][cc] = 0.0;
    const double* qrow[RPW];
    bool live[RPW];
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
      live[q] = (row + q) < w_hi;
      qrow[q] = Q + (int64_t)(live[q] ? row + q : row) * ldq + k0;
    }
    int k = 2 * lane;
#pragma unroll 2
    for (; k < kfull; k += 64) {
      double2 qv[RPW];
#pragma unroll
      for (int q = 0; q < RPW; ++q)
        qv[q] = live[q] ? __ldcs(reinterpret_cast<const double2*>(qrow[q] + k))
                        : make_double2(0.0, 0.0);
#pragma unroll
      for (int cc = 0; cc < R; ++cc) {
        double2 v = *reinterpret_cast<const double2*>(&vt[cc * kc + k]);
#pragma unroll
        for (int q = 0; q < RPW; ++q) acc[q][cc] = fma(qv[q].x, v.x, fma(qv[q].y, v.y, acc[q][cc]));
      }
    }
    // ragged tail (< 64 columns), scalar loads
    for (int kt = kfull + lane; kt < klen; kt += 32) {
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        double qq = live[q] ? qrow[q][kt] : 0.0;
#pragma unroll
        for (int cc = 0; cc < R; ++cc) acc[q][cc] = fma(qq, vt[cc * kc + kt], acc[q][cc]);
      }
    }
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) {
        double v = acc[q][cc];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[q][cc] = v;
      }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < RPW; ++q)
        if (live[q]) {
          double* o = part + ((int64_t)split * nrows + row + q) * R;
#pragma unroll
          for (int cc = 0; cc < R; ++cc) o[cc] = acc[q][cc];
        }
    }
  }
}

// out_full[(row0 + row)·r + c] = Σ_split part[split][row][c]  (fixed order)
__global__ void k_spmm_reduce(const double* __restrict__ part, int nsplit, int nrows, int r,
                              double* __restrict__ out, const int* __restrict__ stop) {
  if (stop && *stop) return;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t tot = (int64_t)nrows * r;
  if (t >= tot) return;
  double s = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) s += part[sp * tot + t];
  out[t] = s;
}

static int rpw_for(int r) { return r == 1 ? 8 : (r <= 6 ? 4 : 2); }
static int kc_for(int r) { return r <= 2 ? 4096 : (r <= 6 ? 1024 : 512); }

SpmmPlan spmm_plan(xm_ctx* c, int r) {
  SpmmPlan p;
  p.rpw = rpw_for(r);
  p.kc = std::min<int>(kc_for(r), (int)round_up(std::max(c->n, 2), 64));
  p.nsplit = ceil_div(c->n, p.kc);
  int smem = r * p.kc * 8;
  int occ = std::max(1, std::min(8, (int)((227 * 1024) / std::max(smem + 1024, 1))));
  int slots = 148 * occ;
  int rows = std::max(c->nrows, 1);
  int maxblk = std::max(1, rows / 8);  // ≥ 1 row per warp
  int waves = 1;
  int nrb = std::max(1, slots * waves / p.nsplit);
  while (nrb > maxblk && nrb > 1) nrb = std::max(1, nrb / 2);
  // aim for ≥ 2 waves when each CTA would stream a lot of rows
  if ((int64_t)rows / nrb > 512 && nrb * 2 <= maxblk) nrb *= 2;
  p.nrowblk = std::min(nrb, maxblk);
  return p;
}

template <int R>
static void launch_partial_r(xm_ctx* c, const double* V, double* part, const SpmmPlan& pl,
                             const int* stop, int* exec) {
  dim3 grid(pl.nrowblk, pl.nsplit);
  size_t smem = (size_t)R * pl.kc * 8;
  auto run = [&](auto kern) {
    static bool attr_set = false;
    if (!attr_set && smem > 48 * 1024) {
      XM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    attr_set = true;
    kern<<<grid, kSpmmThreads, smem, c->stream>>>(c->Q.p, c->ldq, c->nrows, c->n, V, pl.kc,
                                                  pl.nrowblk, part, stop, exec);
  };
  constexpr int RPW = (R == 1) ? 8 : (R <= 6 ? 4 : 2);  // = rpw_for(R)
  if (pl.rpw != RPW) throw Error(XM_EINVAL, "spmm plan / kernel mismatch");
  run(k_spmm_partial<R, RPW>);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void spmm_partial(xm_ctx* c, const double* V, int r, double* part, const SpmmPlan& pl,
                  const int* stop, int* exec) {
  switch (r) {
#define XM_R(RR) case RR: launch_partial_r<RR>(c, V, part, pl, stop, exec); break;
    XM_R(1) XM_R(2) XM_R(3) XM_R(4) XM_R(5) XM_R(6) XM_R(7) XM_R(8) XM_R(9) XM_R(10) XM_R(11)
    XM_R(12)
#undef XM_R
    default: throw Error(XM_EINVAL, "rank r out of range (1..12)");
  }
}

void spmm_reduce(xm_ctx* c, const double* part, int r, const SpmmPlan& pl, double* out_full,
                 const int* stop) {
  int64_t tot = (int64_t)c->nrows * r;
  if (tot == 0) return;
  k_spmm_reduce<<<ceil_div(tot, 256), 256, 0, c->stream>>>(part, pl.nsplit, c->nrows, r,
                                                          out_full + (int64_t)c->row0 * r, stop);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void spmm_full(xm_ctx* c, const double* V, int r, double* out_full, const int* stop) {
  SpmmPlan pl = spmm_plan(c, r);
  c->part.alloc((size_t)pl.nsplit * std::max(c->nrows, 1) * r);
  bool timed = c->opt.profile != 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
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
    e1 = c->ev_pool[c->ev_used++];
    XM_CUDA(cudaEventRecord(e0, c->stream));
  }
  int* exec = nullptr;
  if (timed) {
    size_t pair = c->ev_used / 2 - 1;
    exec = c->ev_exec.p + pair;
    c->ev_bytes[pair] = 8.0 * ((double)c->nrows * c->n + (double)c->n * r + (double)c->nrows * r);
  }
  spmm_partial(c, V, r, c->part.p, pl, stop, exec);
  if (timed) XM_CUDA(cudaEventRecord(e1, c->stream));
  spmm_reduce(c, c->part.p, r, pl, out_full, stop);
  if (c->world > 1) allgather_rows(c, out_full, r);
  c->stats.spmm_calls++;
  c->stats.spmm_rows = c->nrows;
}

// Accumulate the CUDA-event time of every profiled SpMM launch (pairs of events
// recorded on the launching stream around k_spmm_partial) into stats.spmm_ms.
void harvest_events(xm_ctx* c) {
  if (c->ev_used == 0) return;
  XM_CUDA(cudaEventSynchronize(c->ev_pool[c->ev_used - 1]));
  std::vector<int> exec(c->ev_used / 2);
  XM_CUDA(cudaMemcpy(exec.data(), c->ev_exec.p, exec.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (size_t q = 0; q + 1 < c->ev_used; q += 2) {
    if (!exec[q / 2]) continue;  // speculative launch that early-exited (tCG already stopped)
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
