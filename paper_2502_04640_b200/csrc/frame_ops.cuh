// frame_ops.cuh — per-camera (3×r block) device helpers shared by the SpMM
// epilogues and the manifold kernels.  See manifold.cu for the formulas
// (Prop. 5; readings C4, C5 in DESIGN.md).
#pragma once
#include "xm_internal.cuh"

namespace xm {

template <int R>
struct Blk {
  double v[3][R];
};

template <int R>
__device__ __forceinline__ void load_blk(const double* __restrict__ X, int i, Blk<R>& b) {
  const double* p = X + (int64_t)3 * i * R;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) b.v[a][c] = p[a * R + c];
}
template <int R>
__device__ __forceinline__ void store_blk(double* __restrict__ X, int i, const Blk<R>& b) {
  double* p = X + (int64_t)3 * i * R;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) p[a * R + c] = b.v[a][c];
}
// M = A Bᵀ (3×3)
template <int R>
__device__ __forceinline__ void mul_abt(const Blk<R>& A, const Blk<R>& B, double M[3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < R; ++c) s = fma(A.v[a][c], B.v[b][c], s);
      M[a][b] = s;
    }
}
template <int R>
__device__ __forceinline__ double frob2(const Blk<R>& A) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) s = fma(A.v[a][c], A.v[a][c], s);
  return s;
}
template <int R>
__device__ __forceinline__ double dotb(const Blk<R>& A, const Blk<R>& B) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) s = fma(A.v[a][c], B.v[a][c], s);
  return s;
}
// Λ = sym(M) (anchor) or sym₀(M)/α, packed (xx, yy, zz, xy, xz, yz)
__device__ __forceinline__ void sym_lambda(const double M[3][3], bool anchor, double alpha,
                                           double L[6]) {
  double xx = M[0][0], yy = M[1][1], zz = M[2][2];
  double xy = 0.5 * (M[0][1] + M[1][0]);
  double xz = 0.5 * (M[0][2] + M[2][0]);
  double yz = 0.5 * (M[1][2] + M[2][1]);
  if (anchor) {
    L[0] = xx; L[1] = yy; L[2] = zz; L[3] = xy; L[4] = xz; L[5] = yz;
  } else {
    double tr3 = (xx + yy + zz) / 3.0;
    double ia = 1.0 / alpha;
    L[0] = (xx - tr3) * ia; L[1] = (yy - tr3) * ia; L[2] = (zz - tr3) * ia;
    L[3] = xy * ia; L[4] = xz * ia; L[5] = yz * ia;
  }
}
// out = scaleA·A − scaleL·Λ B   (Λ symmetric, packed)
template <int R>
__device__ __forceinline__ void sub_lam(const Blk<R>& A, const double L[6], const Blk<R>& B,
                                        double scaleA, double scaleL, Blk<R>& out) {
  const double Lm[3][3] = {{L[0], L[3], L[4]}, {L[3], L[1], L[5]}, {L[4], L[5], L[2]}};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double s = Lm[a][0] * B.v[0][c] + Lm[a][1] * B.v[1][c] + Lm[a][2] * B.v[2][c];
      out.v[a][c] = scaleA * A.v[a][c] - scaleL * s;
    }
}
// in-place tangent projection of W at Y:  W − sym₀(W Yᵀ) Y / α  (anchor: sym, α = 1)
template <int R>
__device__ __forceinline__ void project_blk(const Blk<R>& Y, bool anchor, Blk<R>& W) {
  double M[3][3], L[6];
  mul_abt<R>(W, Y, M);
  double alpha = anchor ? 1.0 : frob2<R>(Y) / 3.0;
  sym_lambda(M, anchor, alpha, L);
  Blk<R> o;
  sub_lam<R>(W, L, Y, 1.0, 1.0, o);
  W = o;
}

__host__ __device__ constexpr int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

// Fixed-order block reduction of NC components over a block of NT threads →
// partials[blockIdx.x·NC + c].  min_mask bit c ⇒ component c uses min.
template <int NC, int NT>
__device__ __forceinline__ void block_reduce_store(double (&v)[NC], double* __restrict__ partials,
                                                   unsigned min_mask = 0u) {
  __shared__ double sh[NC][NT];
#pragma unroll
  for (int c = 0; c < NC; ++c) sh[c][threadIdx.x] = v[c];
  __syncthreads();
  constexpr int P = pow2_floor(NT);  // largest power of two ≤ NT
  if constexpr (P != NT) {  // fold the tail [P, NT) onto [0, NT − P)
    if (threadIdx.x < NT - P) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double a = sh[c][threadIdx.x], b = sh[c][threadIdx.x + P];
        sh[c][threadIdx.x] = ((min_mask >> c) & 1u) ? fmin(a, b) : a + b;
      }
    }
    __syncthreads();
  }
  for (int s = P / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double a = sh[c][threadIdx.x], b = sh[c][threadIdx.x + s];
        sh[c][threadIdx.x] = ((min_mask >> c) & 1u) ? fmin(a, b) : a + b;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) partials[blockIdx.x * NC + c] = sh[c][0];
  }
  __syncthreads();
}

// Fixed-order sum of nblk partials (stride `stride`, offset `comp`) by a whole
// block of NT threads; every thread returns the same value.  Used to fold the
// scalar tCG control into the vector kernels (each block recomputes the same
// scalar from the same partials in the same order ⇒ identical everywhere).
template <int NT>
__device__ __forceinline__ double block_sum_all(const double* __restrict__ part, int nblk,
                                                int stride = 1, int comp = 0) {
  __shared__ double sh[NT];
  double a = 0.0;
  for (int b = threadIdx.x; b < nblk; b += NT) a += part[b * stride + comp];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}

// Sense-reversing software grid barrier.  Valid only for kernels whose G
// CTAs are all co-resident (one per SM, G ≤ #SMs; launched cooperatively or
// checked on the host) and issued on the library's single stream.
__device__ __forceinline__ void grid_barrier(GridBar* gb, int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile int* vs = &gb->sense;
    const int s = *vs;
    __threadfence();
    if (atomicAdd(&gb->count, 1) == G - 1) {
      gb->count = 0;
      __threadfence();
      atomicExch(&gb->sense, s ^ 1);
    } else {
      while (*vs == s) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Grid barrier on a monotonically increasing 64-bit arrival counter (reset
// to 0 before a launch sequence; every barrier adds G): the last arrival
// itself releases the others — one release-add per CTA and acquire polling of
// one L2 line, no reset / flip round trip.  Same co-residency requirement.
__device__ __forceinline__ void grid_sync(unsigned long long* cnt, unsigned G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long v, cur;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(v) : "l"(cnt) : "memory");
    const unsigned long long target = (v / G + 1) * G;
    do {
      asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(cnt) : "memory");
    } while (cur < target);
  }
  __syncthreads();
}

// Fixed-order block sum for any block size NT (multiple of 32): xor-shuffle
// tree per warp, then warp sums in warp order.  Every thread returns the same
// value, and every block running it on the same inputs gets the same bits.
template <int NT>
__device__ __forceinline__ double block_sum_fixed(double v) {
  static_assert(NT % 32 == 0, "whole warps");
  __shared__ double ws[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = ws[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) t += ws[w];
  __syncthreads();
  return t;
}
// Σ part[0..n) in a fixed order, identical in every block.  L1-bypassing
// loads: the partials were written by other SMs before a grid barrier.
template <int NT>
__device__ __forceinline__ double block_sum_partials(const double* part, int n) {
  double a = 0.0;
  for (int b = threadIdx.x; b < n; b += NT) a += __ldcg(part + b);
  return block_sum_fixed<NT>(a);
}

}  // namespace xm
