// xm2.cu — XM²: "delete the 10% measurements with the
// largest residuals and re-run the XM solver", with SPEC's residual
// definition and never-disconnect rule; the exact
// selection and restoration order are reading C22.
//
// Everything runs on the device over the canonical (landmark, frame)-sorted
// measurement arrays of the last xm_build_Q:
//   k_edge_residuals   res_c = w_c ‖s_i R_i ũ_c + t_i − p_k‖²   (Eq. (3) summand)
//   radix sort         key = ~bits(res) (descending residual), stable over the
//                      canonical index ⇒ ties by (landmark, frame) ascending
//   k_xm2_drop         the first ⌊frac·E⌋ of that order are dropped
//   k_xm2_useful       per frame: kept measurements of landmarks with ≥ 2 kept
//                      measurements; k_xm2_determine (one thread, deficient
//                      frames only) restores their dropped measurements,
//                      smallest residual first, until each has 3 (C22b)
//   k_cc_*_masked      label propagation over the kept measurements
//   k_xm2_restore      one thread: Kruskal over the dropped list backwards
//                      (smallest residual first) until the frames are in one
//                      component — only runs when the kept graph is split
//   k_xm2_prune        restored measurements whose landmark ends with one kept
//                      measurement are dropped again (minimality, C22b)
//   k_xm2_compact      kept measurements (canonical order) → the input arrays
//                      of the rebuild, with their caller-side input indices
#include "xm_internal.cuh"

namespace xm {

__global__ void k_edge_residuals(int64_t E, const int32_t* __restrict__ fr, const int32_t* __restrict__ lm,
                                 const double* __restrict__ pts, const double* __restrict__ w,
                                 const double* __restrict__ Rs, const double* __restrict__ s,
                                 const double* __restrict__ t, const double* __restrict__ p,
                                 double* __restrict__ res) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= E) return;
  const int i = fr[c], k = lm[c];
  const double u0 = pts[3 * c], u1 = pts[3 * c + 1], u2 = pts[3 * c + 2];
  const double* R = Rs + 9 * (int64_t)i;  // row-major R_i (camera → world)
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double x = s[i] * (R[3 * a] * u0 + R[3 * a + 1] * u1 + R[3 * a + 2] * u2) + t[3 * i + a] -
                     p[3 * (int64_t)k + a];
    acc += x * x;
  }
  res[c] = w[c] * acc;
}

// descending residual: residuals are ≥ 0, so their IEEE bits order like the
// values; the complement sorts largest first
__global__ void k_xm2_keys(int64_t E, const double* __restrict__ res, uint64_t* __restrict__ key,
                           uint32_t* __restrict__ val) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= E) return;
  key[c] = ~(uint64_t)__double_as_longlong(res[c]);
  val[c] = (uint32_t)c;
}

__global__ void k_xm2_drop(int64_t E, int64_t nd, const uint32_t* __restrict__ order,
                           int32_t* __restrict__ keep) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= E) return;
  if (j < nd) keep[order[j]] = 0;
}

__global__ void k_xm2_rank(int64_t E, const uint32_t* __restrict__ order, int32_t* __restrict__ rank) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < E) rank[order[j]] = (int32_t)j;
}
__global__ void k_xm2_lmcount(int64_t E, const int32_t* __restrict__ lm, const int32_t* __restrict__ keep,
                              int32_t* __restrict__ kcnt) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < E && keep[e]) atomicAdd(&kcnt[lm[e]], 1);
}
// per frame: 1 if it has fewer than min_obs kept measurements of landmarks with ≥ 2 kept
__global__ void k_xm2_useful(int N, const int32_t* __restrict__ fr_off, const int32_t* __restrict__ fr_edge,
                             const int32_t* __restrict__ lm, const int32_t* __restrict__ keep,
                             const int32_t* __restrict__ kcnt, int min_obs, int32_t* __restrict__ deficient) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int u = 0;
  for (int q = fr_off[i]; q < fr_off[i + 1]; ++q) {
    const int e = fr_edge[q];
    u += (keep[e] && kcnt[lm[e]] >= 2) ? 1 : 0;
  }
  deficient[i] = u < min_obs ? 1 : 0;
}
// one thread: deficient frames in ascending order get dropped measurements
// back, smallest residual (largest drop rank) first, until min_obs useful
__global__ void k_xm2_determine(int N, const int32_t* __restrict__ fr_off, const int32_t* __restrict__ fr_edge,
                                const int32_t* __restrict__ lm, const int32_t* __restrict__ rank,
                                const int32_t* __restrict__ deficient, int min_obs, int32_t* __restrict__ keep,
                                int32_t* __restrict__ restored, int32_t* __restrict__ kcnt) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int i = 0; i < N; ++i) {
    if (!deficient[i]) continue;
    for (;;) {
      int u = 0, best = -1, best_rank = -1;
      for (int q = fr_off[i]; q < fr_off[i + 1]; ++q) {
        const int e = fr_edge[q];
        if (keep[e]) {
          u += kcnt[lm[e]] >= 2 ? 1 : 0;
        } else if (rank[e] > best_rank) {
          best_rank = rank[e];
          best = e;
        }
      }
      if (u >= min_obs || best < 0) break;
      keep[best] = 1;
      restored[best] = 1;
      kcnt[lm[best]] += 1;
    }
  }
}
__global__ void k_xm2_prune(int64_t E, const int32_t* __restrict__ lm, const int32_t* __restrict__ kcnt,
                            const int32_t* __restrict__ restored, int32_t* __restrict__ keep) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < E && restored[e] && keep[e] && kcnt[lm[e]] == 1) keep[e] = 0;
}

__global__ void k_cc_init_m(int n, int32_t* parent) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) parent[v] = v;
}
__global__ void k_cc_hook_m(int64_t E, int N, const int32_t* __restrict__ fr, const int32_t* __restrict__ lm,
                            const int32_t* __restrict__ keep, int32_t* parent, int* changed) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E || !keep[e]) return;
  const int a = parent[fr[e]], b = parent[N + lm[e]];
  if (a != b) {
    atomicMin(&parent[a > b ? a : b], a > b ? b : a);
    *changed = 1;
  }
}
__global__ void k_cc_jump_m(int n, int32_t* parent) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int q = parent[v];
  while (q != parent[q]) q = parent[q];
  parent[v] = q;
}

// Kruskal restoration (reading C22).  label: component root of every node
// after propagation over the kept measurements; uf / hf: scratch (N+M).
// out[0] = restored count, out[1] = frame components left (1 on success).
__global__ void k_xm2_restore(int N, int M, int64_t nd, const int32_t* __restrict__ fr,
                              const int32_t* __restrict__ lm, const uint32_t* __restrict__ order,
                              const int32_t* __restrict__ label, int32_t* __restrict__ uf,
                              uint8_t* __restrict__ hf, int32_t* __restrict__ keep,
                              int32_t* __restrict__ restored_flag, int64_t* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const int n = N + M;
  for (int v = 0; v < n; ++v) {
    uf[v] = label[v];
    hf[v] = 0;
  }
  auto find = [&](int x) {
    while (uf[x] != x) {
      uf[x] = uf[uf[x]];  // path halving
      x = uf[x];
    }
    return x;
  };
  for (int i = 0; i < N; ++i) hf[find(i)] = 1;
  int64_t comps = 0;
  for (int v = 0; v < n; ++v) comps += (uf[v] == v && hf[v]) ? 1 : 0;
  int64_t restored = 0;
  for (int64_t j = nd - 1; j >= 0 && comps > 1; --j) {  // smallest residual first
    const int e = (int)order[j];
    if (keep[e]) continue;  // already back (determined-frame step)
    const int a = find(fr[e]), b = find(N + lm[e]);
    if (a == b) continue;
    const uint8_t fa = hf[a], fb = hf[b];
    uf[b] = a;
    hf[a] = fa | fb;
    keep[e] = 1;
    restored_flag[e] = 1;
    ++restored;
    if (fa && fb) --comps;
  }
  out[0] = restored;
  out[1] = comps;
}

// kept measurements, canonical order → rebuild inputs; caller-side index of
// each (orig == nullptr: the last build's input order is the caller's)
__global__ void k_xm2_compact(int64_t E, const int32_t* __restrict__ keep, const int32_t* __restrict__ pos,
                              const int32_t* __restrict__ fr, const int32_t* __restrict__ lm,
                              const double* __restrict__ pts, const double* __restrict__ w,
                              const int32_t* __restrict__ e_in, const int32_t* __restrict__ orig,
                              int32_t* __restrict__ ofr, int32_t* __restrict__ olm, double* __restrict__ opts,
                              double* __restrict__ ow, int32_t* __restrict__ oorig) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= E || !keep[c]) return;
  const int q = pos[c];
  ofr[q] = fr[c];
  olm[q] = lm[c];
  opts[3 * (int64_t)q] = pts[3 * c];
  opts[3 * (int64_t)q + 1] = pts[3 * c + 1];
  opts[3 * (int64_t)q + 2] = pts[3 * c + 2];
  ow[q] = w[c];
  const int ein = e_in[c];
  oorig[q] = orig ? orig[ein] : ein;
}

// per caller-side measurement: value of canonical measurement c, fill elsewhere
__global__ void k_scatter_user_f64(int64_t E, const double* __restrict__ v, const int32_t* __restrict__ e_in,
                                   const int32_t* __restrict__ orig, double* __restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= E) return;
  const int ein = e_in[c];
  out[orig ? orig[ein] : ein] = v[c];
}
__global__ void k_scatter_user_keep(int64_t E, const int32_t* __restrict__ keep, const int32_t* __restrict__ e_in,
                                    const int32_t* __restrict__ orig, uint8_t* __restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= E) return;
  const int ein = e_in[c];
  out[orig ? orig[ein] : ein] = keep[c] ? 1 : 0;
}
__global__ void k_fill_f64(int64_t n, double v, double* __restrict__ out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) out[j] = v;
}
__global__ void k_fill_i32x(int64_t n, int32_t v, int32_t* __restrict__ out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) out[j] = v;
}

// residuals of the current canonical measurements at the recovered solution
static double* residuals_device(xm_ctx* c) {
  DBuf<double>& res = scratch_f64(c, "xm2_res");
  res.alloc(std::max<int64_t>(c->E, 1));
  const int T = 256;
  k_edge_residuals<<<ceil_div(c->E, T), T, 0, c->stream>>>(c->E, c->e_fr.p, c->e_lm.p, c->e_pts.p, c->e_w.p,
                                                          c->Rs.p, c->s_out.p, c->t_out.p, c->p_out.p, res.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  return res.p;
}

void edge_residuals_user(xm_ctx* c, double* out_dev) {
  const double* res = residuals_device(c);
  const int T = 256;
  k_fill_f64<<<ceil_div(c->E_user, T), T, 0, c->stream>>>(c->E_user, NAN, out_dev);
  k_scatter_user_f64<<<ceil_div(c->E, T), T, 0, c->stream>>>(c->E, res, c->e_in.p,
                                                             c->orig_in.p ? c->orig_in.p : nullptr, out_dev);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
}

void xm2_device(xm_ctx* c, double frac, uint8_t* keep_user_dev, int64_t* n_dropped, int64_t* n_restored) {
  const int T = 256;
  const int64_t E = c->E;
  const int N = c->N, M = c->M;
  const double* res = residuals_device(c);
  // order: residual descending, canonical index ascending on ties
  DBuf<uint64_t>& key = scratch_u64(c, "xm2_key");
  DBuf<uint32_t>& ord = scratch_u32(c, "xm2_ord");
  DBuf<uint64_t>& tk = scratch_u64(c, "sort_tk");
  DBuf<uint32_t>& tv = scratch_u32(c, "sort_tv");
  key.alloc(E);
  ord.alloc(E);
  k_xm2_keys<<<ceil_div(E, T), T, 0, c->stream>>>(E, res, key.p, ord.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  radix_sort_u64(c, key.p, ord.p, E, 64, tk, tv);
  const int64_t nd = (int64_t)std::floor(frac * (double)E);
  DBuf<int32_t>& keep = scratch_i32(c, "xm2_keep");
  keep.alloc(E);
  k_fill_i32x<<<ceil_div(E, T), T, 0, c->stream>>>(E, 1, keep.p);
  k_xm2_drop<<<ceil_div(E, T), T, 0, c->stream>>>(E, nd, ord.p, keep.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  // determined frames (reading C22b)
  constexpr int kMinObs = 3;
  DBuf<int32_t>& rank = scratch_i32(c, "xm2_rank");
  DBuf<int32_t>& restored = scratch_i32(c, "xm2_restored");
  DBuf<int32_t>& kcnt = scratch_i32(c, "xm2_kcnt");
  DBuf<int32_t>& defi = scratch_i32(c, "xm2_deficient");
  rank.alloc(E);
  restored.alloc(E);
  kcnt.alloc(M);
  defi.alloc(N);
  XM_CUDA(cudaMemsetAsync(restored.p, 0, (size_t)E * 4, c->stream));
  XM_CUDA(cudaMemsetAsync(kcnt.p, 0, (size_t)M * 4, c->stream));
  k_xm2_rank<<<ceil_div(E, T), T, 0, c->stream>>>(E, ord.p, rank.p);
  k_xm2_lmcount<<<ceil_div(E, T), T, 0, c->stream>>>(E, c->e_lm.p, keep.p, kcnt.p);
  k_xm2_useful<<<ceil_div(N, T), T, 0, c->stream>>>(N, c->fr_off.p, c->fr_edge.p, c->e_lm.p, keep.p, kcnt.p,
                                                   kMinObs, defi.p);
  k_xm2_determine<<<1, 1, 0, c->stream>>>(N, c->fr_off.p, c->fr_edge.p, c->e_lm.p, rank.p, defi.p, kMinObs,
                                          keep.p, restored.p, kcnt.p);
  XM_CHECK_LAUNCH();
  count_launch(c, 4);
  // connectivity of the kept graph (frames ∪ landmarks), then restoration
  DBuf<int32_t>& label = scratch_i32(c, "xm2_label");
  label.alloc(N + M);
  k_cc_init_m<<<ceil_div(N + M, T), T, 0, c->stream>>>(N + M, label.p);
  count_launch(c);
  int* d_changed = c->flags.p + 8;
  for (int it = 0; it < 100000; ++it) {
    XM_CUDA(cudaMemsetAsync(d_changed, 0, 4, c->stream));
    k_cc_hook_m<<<ceil_div(E, T), T, 0, c->stream>>>(E, N, c->e_fr.p, c->e_lm.p, keep.p, label.p, d_changed);
    k_cc_jump_m<<<ceil_div(N + M, T), T, 0, c->stream>>>(N + M, label.p);
    XM_CHECK_LAUNCH();
    count_launch(c, 2);
    int ch = 0;
    XM_CUDA(cudaMemcpyAsync(&ch, d_changed, 4, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (!ch) break;
  }
  DBuf<int32_t>& uf = scratch_i32(c, "xm2_uf");
  DBuf<uint32_t>& hf = scratch_u32(c, "xm2_hf");
  uf.alloc(N + M);
  hf.alloc((N + M + 3) / 4 + 1);
  DBuf<uint64_t>& outb = scratch_u64(c, "xm2_out");
  outb.alloc(2);
  k_xm2_restore<<<1, 1, 0, c->stream>>>(N, M, nd, c->e_fr.p, c->e_lm.p, ord.p, label.p, uf.p,
                                        reinterpret_cast<uint8_t*>(hf.p), keep.p, restored.p,
                                        reinterpret_cast<int64_t*>(outb.p));
  XM_CHECK_LAUNCH();
  count_launch(c);
  int64_t h_out[2] = {0, 0};
  XM_CUDA(cudaMemcpyAsync(h_out, outb.p, 16, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (h_out[1] != 1) throw Error(XM_EDISCONNECTED, "XM²: graph disconnected even with every measurement");
  // minimality: restored leaves go again
  XM_CUDA(cudaMemsetAsync(kcnt.p, 0, (size_t)M * 4, c->stream));
  k_xm2_lmcount<<<ceil_div(E, T), T, 0, c->stream>>>(E, c->e_lm.p, keep.p, kcnt.p);
  k_xm2_prune<<<ceil_div(E, T), T, 0, c->stream>>>(E, c->e_lm.p, kcnt.p, restored.p, keep.p);
  XM_CHECK_LAUNCH();
  count_launch(c, 2);
  const int32_t* orig = c->orig_in.p ? c->orig_in.p : nullptr;
  if (keep_user_dev) {
    XM_CUDA(cudaMemsetAsync(keep_user_dev, 0, (size_t)c->E_user, c->stream));
    k_scatter_user_keep<<<ceil_div(E, T), T, 0, c->stream>>>(E, keep.p, c->e_in.p, orig, keep_user_dev);
    XM_CHECK_LAUNCH();
    count_launch(c);
  }
  // compact the kept measurements and rebuild Q from them
  DBuf<int32_t>& pos = scratch_i32(c, "xm2_pos");
  pos.alloc(E);
  int32_t* d_total = c->flags.p + 4;
  exclusive_scan_i32(c, keep.p, pos.p, E, d_total);
  int32_t Ek = 0;
  XM_CUDA(cudaMemcpyAsync(&Ek, d_total, 4, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (n_dropped) *n_dropped = E - Ek;
  if (n_restored) *n_restored = nd - (E - Ek);
  DBuf<int32_t>& nfr = scratch_i32(c, "xm2_fr");
  DBuf<int32_t>& nlm = scratch_i32(c, "xm2_lm");
  DBuf<double>& npts = scratch_f64(c, "xm2_pts");
  DBuf<double>& nw = scratch_f64(c, "xm2_w");
  DBuf<int32_t>& norig = scratch_i32(c, "xm2_orig");
  nfr.alloc(Ek);
  nlm.alloc(Ek);
  npts.alloc(3 * (int64_t)Ek);
  nw.alloc(Ek);
  norig.alloc(Ek);
  k_xm2_compact<<<ceil_div(E, T), T, 0, c->stream>>>(E, keep.p, pos.p, c->e_fr.p, c->e_lm.p, c->e_pts.p, c->e_w.p,
                                                     c->e_in.p, orig, nfr.p, nlm.p, npts.p, nw.p, norig.p);
  XM_CHECK_LAUNCH();
  count_launch(c);
  // from here the context's measurement mapping and data matrix are replaced
  // step by step: a failure (e.g. XM_ENOMEM) leaves no consistent previous
  // stage to fall back to, so the context drops to "no data" (stage 0) and a
  // later call must rebuild (xm.h: xm_xm2 error behaviour)
  try {
    c->orig_in.alloc(std::max<int32_t>(Ek, 1));
    XM_CUDA(cudaMemcpyAsync(c->orig_in.p, norig.p, (size_t)Ek * 4, cudaMemcpyDeviceToDevice, c->stream));
    build_Q_device(c, N, M, Ek, nfr.p, nlm.p, npts.p, nw.p);
  } catch (...) {
    c->stage = 0;
    throw;
  }
}

}  // namespace xm
