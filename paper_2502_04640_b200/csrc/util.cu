// util.cu — deterministic reductions, exclusive scan, stable LSD radix sort,
// host/device copy helpers.  All reductions use a fixed grid and a fixed
// combination order, so reruns are bitwise identical.
#include "xm_internal.cuh"

namespace xm {

void ensure_smem_attr(const void* kern, size_t smem) {
  thread_local std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  XM_CUDA(cudaGetDevice(&dev));
  size_t& cur = done[{kern, dev}];
  if (smem > cur) {
    XM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void copy_in(xm_ctx* c, void* dst_dev, const void* src, size_t bytes) {
  if (!bytes) return;
  XM_CUDA(cudaMemcpyAsync(dst_dev, src, bytes,
                          is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                          c->stream));
}

void copy_out(xm_ctx* c, void* dst, const void* src_dev, size_t bytes) {
  if (!bytes || !dst) return;
  bool dev = is_device_ptr(dst);
  XM_CUDA(cudaMemcpyAsync(dst, src_dev, bytes,
                          dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  if (!dev) XM_CUDA(cudaStreamSynchronize(c->stream));
}

void sync(xm_ctx* c) { XM_CUDA(cudaStreamSynchronize(c->stream)); }

// ------------------------------------------------------------------ reduce
// partials: nblk × ncomp (row-major).  One block per component; fixed tree.
__global__ void k_reduce_partials(const double* __restrict__ part, int nblk, int ncomp,
                                  double* __restrict__ out, unsigned min_mask) {
  __shared__ double sh[256];
  int comp = blockIdx.x;
  bool is_min = (min_mask >> comp) & 1u;
  double acc = is_min ? 1.0e300 : 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    double v = part[(int64_t)b * ncomp + comp];
    acc = is_min ? fmin(acc, v) : acc + v;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      sh[threadIdx.x] = is_min ? fmin(sh[threadIdx.x], sh[threadIdx.x + s])
                               : sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[comp] = sh[0];
}

void reduce_partials(xm_ctx* c, const double* partials, int nblk, int ncomp, double* out,
                     unsigned min_mask) {
  k_reduce_partials<<<ncomp, 256, 0, c->stream>>>(partials, nblk, ncomp, out, min_mask);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

// ------------------------------------------------------------------ dot
__global__ void k_dot_flat(const double* __restrict__ a, const double* __restrict__ b, int64_t len,
                           double* __restrict__ partials) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(a[i], b[i], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

// two dot products in one pass (same per-pair arithmetic and order as two
// k_dot_flat launches): partials[blk·2 + q] = block sum of ⟨a_q, b_q⟩
__global__ void k_dot2_flat(const double* __restrict__ a0, const double* __restrict__ b0,
                            const double* __restrict__ a1, const double* __restrict__ b1, int64_t len,
                            double* __restrict__ partials) {
  __shared__ double sh[2][256];
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    acc0 = fma(a0[i], b0[i], acc0);
    acc1 = fma(a1[i], b1[i], acc1);
  }
  sh[0][threadIdx.x] = acc0;
  sh[1][threadIdx.x] = acc1;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + s];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = sh[0][0];
    partials[2 * blockIdx.x + 1] = sh[1][0];
  }
}

void dot2_flat(xm_ctx* c, const double* a0, const double* b0, const double* a1, const double* b1,
               int64_t len, double* partials, int nblk) {
  k_dot2_flat<<<nblk, 256, 0, c->stream>>>(a0, b0, a1, b1, len, partials);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

void dot_flat(xm_ctx* c, const double* a, const double* b, int64_t len, double* partials,
              int nblk) {
  k_dot_flat<<<nblk, 256, 0, c->stream>>>(a, b, len, partials);
  XM_CHECK_LAUNCH();
  count_launch(c);
}

// ------------------------------------------------------------------ scan (int32)
constexpr int kScanItems = 4;
constexpr int kScanThreads = 256;
constexpr int kScanTile = kScanItems * kScanThreads;

__global__ void k_scan_tile(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                            int32_t* __restrict__ block_sums) {
  __shared__ int32_t sh[kScanThreads];
  int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int32_t v[kScanItems];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0;
    s += v[i];
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  // Hillis–Steele inclusive scan of thread sums
  for (int off = 1; off < kScanThreads; off <<= 1) {
    int32_t t = (threadIdx.x >= off) ? sh[threadIdx.x - off] : 0;
    __syncthreads();
    sh[threadIdx.x] += t;
    __syncthreads();
  }
  int32_t run = sh[threadIdx.x] - s;  // exclusive
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == kScanThreads - 1 && block_sums) block_sums[blockIdx.x] = sh[threadIdx.x];
}

__global__ void k_scan_add(int32_t* __restrict__ out, int64_t n,
                           const int32_t* __restrict__ block_off) {
  int64_t i = (int64_t)blockIdx.x * kScanTile + threadIdx.x;
  int32_t add = block_off[blockIdx.x];
  for (int k = 0; k < kScanItems; ++k, i += kScanThreads)
    if (i < n) out[i] += add;
}

__global__ void k_scan_total(const int32_t* in, const int32_t* out, int64_t n, int32_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *total = (n > 0) ? out[n - 1] + in[n - 1] : 0;
}

static void scan_rec(xm_ctx* c, const int32_t* in, int32_t* out, int64_t n, int level = 0) {
  int nb = ceil_div(n, kScanTile);
  if (nb <= 1) {
    k_scan_tile<<<1, kScanThreads, 0, c->stream>>>(in, out, n, nullptr);
    XM_CHECK_LAUNCH();
    count_launch(c);
    return;
  }
  DBuf<int32_t>& sums = scratch_i32(c, "scan_sums" + std::to_string(level));
  DBuf<int32_t>& offs = scratch_i32(c, "scan_offs" + std::to_string(level));
  sums.alloc(nb);
  offs.alloc(nb);
  k_scan_tile<<<nb, kScanThreads, 0, c->stream>>>(in, out, n, sums.p);
  XM_CHECK_LAUNCH();
  scan_rec(c, sums.p, offs.p, nb, level + 1);
  k_scan_add<<<nb, kScanThreads, 0, c->stream>>>(out, n, offs.p);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
}

void exclusive_scan_i32(xm_ctx* c, const int32_t* in, int32_t* out, int64_t n, int32_t* total_dev) {
  if (n <= 0) return;
  if (in == out) {
    DBuf<int32_t>& tmp = scratch_i32(c, "scan_inplace");
    tmp.alloc(n);
    XM_CUDA(cudaMemcpyAsync(tmp.p, in, n * 4, cudaMemcpyDeviceToDevice, c->stream));
    scan_rec(c, tmp.p, out, n);
    if (total_dev) {
      k_scan_total<<<1, 1, 0, c->stream>>>(tmp.p, out, n, total_dev);
      count_launch(c);
    }
    XM_CUDA(cudaStreamSynchronize(c->stream));
    return;
  }
  scan_rec(c, in, out, n);
  if (total_dev) {
    k_scan_total<<<1, 1, 0, c->stream>>>(in, out, n, total_dev);
    XM_CHECK_LAUNCH();
    count_launch(c);
  }
}

// ------------------------------------------------------------------ radix sort
// Stable LSD radix sort of (uint64 key, uint32 value), 8-bit digits.
// Per pass: (1) per-tile digit histogram (digit-major: hist[d·ntiles + t]);
// (2) exclusive scan ⇒ global base of every (digit, tile); (3) stable scatter:
// within a tile, items are ranked in index order with warp match + per-warp
// digit counts, so equal digits keep their input order.
constexpr int kSortThreads = 256;
constexpr int kSortTile = 2048;  // items per tile (8 rounds of 256)

__global__ void k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift, int ntiles,
                             int32_t* __restrict__ hist) {
  __shared__ int32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += kSortThreads) {
    int64_t idx = base + i;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void k_radix_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                int64_t n, int shift, int ntiles, const int32_t* __restrict__ offs,
                                uint64_t* __restrict__ okeys, uint32_t* __restrict__ ovals) {
  __shared__ int32_t base[256];
  __shared__ int32_t running[256];
  __shared__ int32_t wcnt[kSortThreads / 32][256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  base[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
  running[tid] = 0;
  for (int w = 0; w < kSortThreads / 32; ++w) wcnt[w][tid] = 0;
  __syncthreads();
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int round = 0; round < kSortTile / kSortThreads; ++round) {
    int64_t idx = (int64_t)blockIdx.x * kSortTile + round * kSortThreads + tid;
    bool valid = idx < n;
    uint64_t k = valid ? keys[idx] : 0;
    int d = valid ? (int)((k >> shift) & 255) : 256 + lane;  // invalid lanes are unique
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & lt_mask);
    if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      int pre = 0;
      for (int w = 0; w < warp; ++w) pre += wcnt[w][d];
      int pos = base[d] + running[d] + pre + rank;
      okeys[pos] = k;
      ovals[pos] = vals[idx];
    }
    __syncthreads();
    int tot = 0;
    for (int w = 0; w < kSortThreads / 32; ++w) {
      tot += wcnt[w][tid];
      wcnt[w][tid] = 0;
    }
    running[tid] += tot;
    __syncthreads();
  }
}

void radix_sort_u64(xm_ctx* c, uint64_t* keys, uint32_t* vals, int64_t n, int bits,
                    DBuf<uint64_t>& tmp_k, DBuf<uint32_t>& tmp_v) {
  if (n <= 1) return;
  int ntiles = ceil_div(n, kSortTile);
  tmp_k.alloc(n);
  tmp_v.alloc(n);
  DBuf<int32_t>& hist = scratch_i32(c, "radix_hist");
  DBuf<int32_t>& offs = scratch_i32(c, "radix_offs");
  hist.alloc((size_t)256 * ntiles);
  offs.alloc((size_t)256 * ntiles);
  uint64_t *ka = keys, *kb = tmp_k.p;
  uint32_t *va = vals, *vb = tmp_v.p;
  int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    int shift = 8 * p;
    k_radix_hist<<<ntiles, kSortThreads, 0, c->stream>>>(ka, n, shift, ntiles, hist.p);
    XM_CHECK_LAUNCH();
    count_launch(c);
    exclusive_scan_i32(c, hist.p, offs.p, (int64_t)256 * ntiles, nullptr);
    k_radix_scatter<<<ntiles, kSortThreads, 0, c->stream>>>(ka, va, n, shift, ntiles, offs.p, kb, vb);
    XM_CHECK_LAUNCH();
    count_launch(c);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != keys) {
    XM_CUDA(cudaMemcpyAsync(keys, ka, n * 8, cudaMemcpyDeviceToDevice, c->stream));
    XM_CUDA(cudaMemcpyAsync(vals, va, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  }
  XM_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace xm
