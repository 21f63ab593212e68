// xm_api.cu — the C ABI (include/xm.h) and the host-side control of
// Algorithm 1 (Riemannian staircase) with the Riemannian
// trust-region / truncated-CG local optimiser.
//
// The host only holds O(1) scalars per iteration (TR radius, ρ) and the k
// Lanczos coefficients; every O(n) and O(n²) operation is a device kernel.
// The tCG inner loop runs from device-resident state (TcgState): kernels read
// α, β, τ and the stop flag from device memory, so the host launches tCG
// iterations in batches and synchronises once per batch.
#include "xm_internal.cuh"

#include <algorithm>

#include <chrono>
#include <cmath>
#include <cstring>

using namespace xm;

namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

template <typename F>
xm_status guard(xm_ctx* c, F&& f) {
  try {
    if (c) XM_CUDA(cudaSetDevice(c->device));
    f();
    return XM_OK;
  } catch (const Error& e) {
    if (c) c->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->last_error = e.what();
    return XM_ECUDA;
  }
}

void require_stage(xm_ctx* c, int stage) {
  if (c->stage < stage) throw Error(XM_ESTATE, "call order violated");
}

constexpr int kMaxCols = XM_MAX_R + 1;

void alloc_vectors(xm_ctx* c) {
  int64_t rows = std::max<int64_t>(c->n, (int64_t)c->world * 3 * c->nfpr);
  rows = round_up(rows, 32);
  if (c->n_alloc == rows && c->Y.p) return;
  c->n_alloc = rows;
  size_t sz = (size_t)rows * kMaxCols + 64;
  for (DBuf<double>* b : {&c->Y, &c->QY, &c->grad, &c->eta, &c->Heta, &c->res, &c->dir, &c->Hdir,
                          &c->Ynew, &c->Dv, &c->QD, &c->tmp, &c->tmp2, &c->hY, &c->hV, &c->hO,
                          &c->hQY}) {
    b->alloc(sz);
    XM_CUDA(cudaMemsetAsync(b->p, 0, sz * 8, c->stream));
  }
  c->lam.alloc((size_t)c->N * 6 + 6);
  c->scal.alloc(64);
  c->tcg.alloc(2);
  c->flags.alloc(16);
  c->cert_v.alloc((size_t)rows + 64);
  c->red.alloc((size_t)ceil_div(c->N, 128) * 4 + 1024);
  c->part1.alloc(4096);   // fixed addresses: captured by the tCG graphs
  c->part2.alloc((size_t)ceil_div(c->N, 128) + 4096);
}

void read_scal(xm_ctx* c, int first, int count, double* out) {
  XM_CUDA(cudaMemcpyAsync(out, c->scal.p + first, count * 8, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
}

// QY = Q·Y, Λ, grad, and scal_out[0..2] = f, ‖g‖², min α  (fused on one GPU)
void grad_fused(xm_ctx* c, int r, const double* Y, double* QY, double* grad, double* scal_out) {
  if (fused_epilogues(c)) {
    c->part1.alloc(2048);
    SpmmEpiArgs ep{};
    ep.out = QY;
    ep.out2 = grad;
    ep.lam_out = c->lam.p;
    ep.partials = c->part1.p;
    spmm(c, Y, r, EPI_GRAD, ep);
    reduce_partials(c, c->part1.p, spmm_grid(c, r), 3, scal_out, 4u);
  } else {
    spmm_full(c, Y, r, QY, nullptr);
    grad_and_multipliers(c, r, Y, QY, grad, scal_out);
  }
}

// fresh QY and gradient at c->Y; returns f, ‖g‖², α_min
void eval_point(xm_ctx* c, double* f, double* g2, double* amin) {
  grad_fused(c, c->r, c->Y.p, c->QY.p, c->grad.p, c->scal.p);
  double h[3];
  read_scal(c, 0, 3, h);
  *f = h[0];
  *g2 = h[1];
  *amin = h[2];
}

// D ↦ (QD, ⟨QY, D⟩, ⟨D, QD⟩) → scal_out[0..1]
void df_product(xm_ctx* c, int r, const double* D, const double* QY, double* QD, double* scal_out) {
  const int64_t len = (int64_t)c->n * r;
  if (dense_fused(c)) {
    c->part2.alloc(4096);
    SpmmEpiArgs ep{};
    ep.out = QD;
    ep.aux = QY;
    ep.partials = c->part2.p;
    spmm(c, D, r, EPI_DF, ep);
    reduce_partials(c, c->part2.p, spmm_grid(c, r), 2, scal_out);
  } else {
    spmm_full(c, D, r, QD, nullptr);
    c->lz_part.alloc((size_t)kDotBlocks * 4 + 64);
    dot2_flat(c, QY, D, D, QD, len, c->lz_part.p, kDotBlocks);  // ⟨QY, D⟩, ⟨D, QD⟩
    reduce_partials(c, c->lz_part.p, kDotBlocks, 2, scal_out);
  }
}

// ⟨a_q, b_q⟩ for up to 4 pairs of flat arrays of length len → host
void dots(xm_ctx* c, int64_t len, int npair, const double* const* a, const double* const* b,
          double* out) {
  c->lz_part.alloc((size_t)kDotBlocks * 4 + 64);
  for (int q = 0; q < npair; ++q) {
    dot_flat(c, a[q], b[q], len, c->lz_part.p, kDotBlocks);
    reduce_partials(c, c->lz_part.p, kDotBlocks, 1, c->scal.p + 8 + q);
  }
  read_scal(c, 8, npair, out);
}

// Capture `tcg_batch` tCG iterations at rank r into a CUDA graph (once; all
// buffers used by the iteration have fixed addresses).  Every kernel in it
// early-exits once the device-side tCG state says stop, so a replay past the
// end of tCG is a cheap no-op.  With profile=1 each SpMM is bracketed by event
// nodes owned by the graph (harvested after every replay).
uintptr_t reg_bits(xm_ctx* c) {
  uint64_t b;
  std::memcpy(&b, &c->opt.scale_reg, 8);
  return (uintptr_t)b;
}

std::vector<uintptr_t> graph_signature(xm_ctx* c) {
  return {(uintptr_t)c->N, (uintptr_t)c->n, (uintptr_t)c->ldq, (uintptr_t)c->Q.p,
          (uintptr_t)c->Y.p, (uintptr_t)c->dir.p, (uintptr_t)c->lam.p, (uintptr_t)c->tcg.p,
          (uintptr_t)c->part1.p, (uintptr_t)c->part2.p, (uintptr_t)c->opt.profile,
          (uintptr_t)c->f0, (uintptr_t)c->f1, (uintptr_t)c->sym_part.p, (uintptr_t)c->gbar.p,
          (uintptr_t)c->sym_plan, (uintptr_t)c->gsync.p, (uintptr_t)c->fused_tcg,
          (uintptr_t)c->opt.spmm_kernel, reg_bits(c), (uintptr_t)c->implicit_active,
          (uintptr_t)c->Kinv.p, (uintptr_t)c->imp_lm.p, (uintptr_t)c->e_fr.p,
          (uintptr_t)c->imp_pts.p, (uintptr_t)c->imp_mom.p, (uintptr_t)c->imp_tb.p,
          (uintptr_t)c->imp_sym_part.p, (uintptr_t)c->imp_sym_plan,
          // the matrix-free kernels take E / M by value (array offsets, loop
          // bounds): an XM² rebuild at the same addresses must recapture
          (uintptr_t)c->E, (uintptr_t)c->M, (uintptr_t)c->imp_k0, (uintptr_t)c->imp_k1,
          (uintptr_t)c->imp_f0, (uintptr_t)c->imp_f1, (uintptr_t)c->imp_ka, (uintptr_t)c->imp_kb};
}

void destroy_graph(xm_ctx::TcgGraph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  for (cudaEvent_t e : g.ev) cudaEventDestroy(e);
  g.exec = nullptr;
  g.ev.clear();
  g.bytes.clear();
  g.sig.clear();
  g.batch = 0;
  g.loop = false;
}

// The whole tCG loop as ONE graph launch: a conditional WHILE node whose body
// is one three-kernel iteration (product + HVP epilogue, k_tcg_update,
// k_tcg_dir); k_tcg_dir clears the condition when the device state says stop,
// so no iteration past the stop is launched and the host syncs once per tCG
// solve instead of once per batch.  Profiling runs keep the batched graphs
// (event-record nodes are not allowed in conditional bodies).  Returns false
// (nothing built) where unsupported.
static bool capture_tcg_loop(xm_ctx* c, int r, xm_ctx::TcgGraph& g) {
  if (c->opt.profile || tcg_fused_supported(c, r) || std::getenv("XM_NO_COND_GRAPH")) return false;
  cudaGraph_t graph = nullptr;
  XM_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle h = 0;
  cudaGraph_t body = nullptr;
  cudaGraphNode_t node = nullptr;
  if (cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(graph);
    return false;
  }
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  if (cudaGraphAddNode(&node, graph, nullptr, 0, &cp) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(graph);
    return false;
  }
  body = cp.conditional.phGraph_out[0];
  cudaStream_t orig = c->stream;
  const int64_t l0 = c->stats.kernel_launches, s0 = c->stats.spmm_calls;
  c->stream = c->cap_stream;
  c->cap_cond = h;
  c->cap_cond_on = true;
  bool ok = true;
  try {
    XM_CUDA(cudaStreamBeginCaptureToGraph(c->cap_stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed));
    tcg_iteration(c, r);
    cudaGraph_t out = nullptr;
    XM_CUDA(cudaStreamEndCapture(c->cap_stream, &out));
  } catch (...) {
    cudaGraph_t out = nullptr;
    cudaStreamEndCapture(c->cap_stream, &out);
    cudaGetLastError();
    ok = false;
  }
  c->stream = orig;
  c->cap_cond_on = false;
  c->cap_cond = 0;
  g.launches = c->stats.kernel_launches - l0;
  g.spmms = c->stats.spmm_calls - s0;
  c->stats.kernel_launches = l0;
  c->stats.spmm_calls = s0;
  if (ok && cudaGraphInstantiate(&g.exec, graph, 0) != cudaSuccess) {
    cudaGetLastError();
    g.exec = nullptr;
    ok = false;
  }
  cudaGraphDestroy(graph);
  if (!ok) return false;
  g.loop = true;
  g.batch = 0;
  return true;
}

xm_ctx::TcgGraph* tcg_graph(xm_ctx* c, int r) {
  auto& g = c->tcg_graphs[r];
  auto sig = graph_signature(c);
  if (g.exec && g.sig == sig) return &g;
  destroy_graph(g);
  g.sig = sig;
  if (!c->cap_stream) XM_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  sync(c);
  if (capture_tcg_loop(c, r, g)) return &g;
  g.batch = c->tcg_batch;
  g.execf.alloc((size_t)g.batch * 4 + 8);
  XM_CUDA(cudaMemsetAsync(g.execf.p, 0, g.execf.n * sizeof(int), c->stream));
  sync(c);
  cudaStream_t orig = c->stream;
  const int64_t l0 = c->stats.kernel_launches, s0 = c->stats.spmm_calls;
  c->stream = c->cap_stream;
  c->cap_target = &g;
  cudaGraph_t graph = nullptr;
  try {
    XM_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
    if (c->opt.profile)
      XM_CUDA(cudaMemsetAsync(g.execf.p, 0, g.execf.n * sizeof(int), c->cap_stream));
    for (int b = 0; b < g.batch; ++b) tcg_iteration(c, r);
    XM_CUDA(cudaStreamEndCapture(c->cap_stream, &graph));
  } catch (...) {
    cudaStreamEndCapture(c->cap_stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    c->stream = orig;
    c->cap_target = nullptr;
    throw;
  }
  c->stream = orig;
  c->cap_target = nullptr;
  g.launches = c->stats.kernel_launches - l0;
  g.spmms = c->stats.spmm_calls - s0;
  c->stats.kernel_launches = l0;
  c->stats.spmm_calls = s0;
  XM_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
  cudaGraphDestroy(graph);
  return &g;
}

void harvest_graph(xm_ctx* c, xm_ctx::TcgGraph& g) {
  const size_t np = g.bytes.size();
  if (!np) return;
  std::vector<int> ex(np);
  XM_CUDA(cudaMemcpy(ex.data(), g.execf.p, np * sizeof(int), cudaMemcpyDeviceToHost));
  for (size_t q = 0; q < np; ++q) {
    if (!ex[q]) continue;
    float ms = 0.f;
    XM_CUDA(cudaEventElapsedTime(&ms, g.ev[2 * q], g.ev[2 * q + 1]));
    c->stats.spmm_ms += ms;
    c->stats.spmm_timed++;
    c->stats.spmm_alg_bytes += g.bytes[q];
  }
}

// XM_PHASES diagnostics: lap(k) adds the time since the previous lap to slot k.
struct PhaseClock {
  xm_ctx* c;
  double t = 0.0;
  explicit PhaseClock(xm_ctx* cc) : c(cc) {
    if (c->phases_on) {
      sync(c);
      t = now_ms();
    }
  }
  void lap(int k) {
    if (!c->phases_on) return;
    sync(c);
    const double n = now_ms();
    c->phase_ms[k] += n - t;
    c->phase_n[k]++;
    t = n;
  }
};
static const char* kPhaseNames[8] = {"tcg", "retract+df", "accept+grad", "eval_point",
                                     "certify", "escape", "lanczos", "cholesky"};

// One Steihaug–Toint tCG solve (O5) at the current c->Y, c->grad, c->lam (the
// last gradient pass) with radius Delta; returns the final device state
// (η in c->eta, Hη in c->Heta).  Path: the whole loop in one cooperative
// launch (tcg_persist.cu) when supported, else CUDA-graph batches of
// iterations (fused or three-kernel, manifold.cu).
// defer (conditional-graph path only): the final state is copied into the
// pinned host scalars without a sync and *deferred is set; the caller reads it
// after its next sync (tcg_deferred_state) — one host round trip per outer
// iteration instead of three.
TcgState run_tcg(xm_ctx* c, int r, double Delta, bool* deferred = nullptr) {
  tcg_init(c, r, Delta);
  TcgState hs{};
  if (deferred) *deferred = false;
  const bool persist = tcg_persist_supported(c, r);
  xm_ctx::TcgGraph* g = !persist && c->use_graphs && c->world == 1 ? tcg_graph(c, r) : nullptr;
  if (persist) {  // the whole tCG loop in one cooperative launch (tcg_persist.cu)
    const bool timed = c->opt.profile != 0;
    if (timed && !c->ev_persist[0]) {
      XM_CUDA(cudaEventCreate(&c->ev_persist[0]));
      XM_CUDA(cudaEventCreate(&c->ev_persist[1]));
    }
    if (timed) XM_CUDA(cudaEventRecord(c->ev_persist[0], c->stream));
    tcg_persist_launch(c, r);
    if (timed) XM_CUDA(cudaEventRecord(c->ev_persist[1], c->stream));
    XM_CUDA(cudaMemcpyAsync(&hs, c->tcg.p, sizeof(TcgState), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    c->stats.spmm_calls += hs.n_hvp;
    if (timed && hs.n_hvp > 0) {  // per-iteration figures: one Q stream per iteration
      float ms = 0.f;
      XM_CUDA(cudaEventElapsedTime(&ms, c->ev_persist[0], c->ev_persist[1]));
      c->stats.spmm_ms += ms;
      c->stats.spmm_timed += hs.n_hvp;
      c->stats.spmm_alg_bytes += hs.n_hvp * tcg_persist_bytes_per_iter(c, r);
    }
  }
  const int64_t s0 = c->stats.spmm_calls;
  while (!persist) {
    if (g && g->loop) {  // the whole loop in one launch (the condition ends it)
      XM_CUDA(cudaGraphLaunch(g->exec, c->stream));
      if (deferred && c->hpin) {
        XM_CUDA(cudaMemcpyAsync(c->hpin + kPinTcg, c->tcg.p, sizeof(TcgState), cudaMemcpyDeviceToHost,
                                c->stream));
        c->tcg_defer_launches = g->launches;
        *deferred = true;
        return hs;
      }
      XM_CUDA(cudaMemcpyAsync(&hs, c->tcg.p, sizeof(TcgState), cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      // iterations launched: one per HVP plus the final one whose update saw the stop
      c->stats.kernel_launches += g->launches * std::max<int64_t>(1, hs.n_hvp);
      if (!hs.stop) throw Error(XM_ECUDA, "tCG loop graph returned before its stop");
      c->stats.spmm_calls = s0 + hs.n_hvp;
      break;
    } else if (g) {
      XM_CUDA(cudaGraphLaunch(g->exec, c->stream));
      c->stats.kernel_launches += g->launches;
    } else {
      for (int b = 0; b < c->tcg_batch; ++b) tcg_iteration(c, r);
    }
    XM_CUDA(cudaMemcpyAsync(&hs, c->tcg.p, sizeof(TcgState), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (g && c->opt.profile) harvest_graph(c, *g);
    if (hs.stop) {
      // products that actually ran (batched iterations after the stop exit early)
      c->stats.spmm_calls = s0 + hs.n_hvp;
      break;
    }
  }
  return hs;
}

// the state of a deferred conditional-graph tCG, after the caller's sync
TcgState tcg_deferred_state(xm_ctx* c) {
  TcgState hs;
  std::memcpy(&hs, c->hpin + kPinTcg, sizeof(TcgState));
  c->stats.kernel_launches += c->tcg_defer_launches * std::max<int64_t>(1, hs.n_hvp);
  if (!hs.stop) throw Error(XM_ECUDA, "tCG loop graph returned before its stop");
  c->stats.spmm_calls += hs.n_hvp;  // graph replays do not count products host-side
  return hs;
}

// The outer iteration's step after tCG: retraction of η (+ ⟨g,η⟩, ⟨η,Hη⟩ into
// scal[10..11]), the cancellation-free Δf product (scal[8..9]) and the App. D
// term.  One GPU with profiling off: replayed as ONE cached graph per rank
// (the same kernels in the same order — bitwise the same results — minus the
// per-kernel launch latencies).
static void post_tcg_sequence(xm_ctx* c, int r) {
  XM_CUDA(cudaMemsetAsync(c->flags.p, 0, sizeof(int), c->stream));
  const int nb = frame_blocks(c);
  retract(c, r, c->Y.p, c->eta.p, 1.0, c->Ynew.p, c->Dv.p, c->flags.p, c->grad.p, c->Heta.p, c->red.p);
  reduce_partials(c, c->red.p, nb, 2, c->scal.p + 10);
  df_product(c, r, c->Dv.p, c->QY.p, c->QD.p, c->scal.p + 8);
  if (c->opt.scale_reg != 0.0) reg_frames(c, r, c->Y.p, c->Dv.p, c->scal.p + 24);
}

static void post_tcg(xm_ctx* c, int r) {
  const int nb = frame_blocks(c);
  c->red.alloc((size_t)nb * 4 + 1024);
  if (c->opt.profile || !c->use_graphs || c->world != 1 || std::getenv("XM_NO_POST_GRAPH")) {
    post_tcg_sequence(c, r);
    return;
  }
  auto& g = c->post_graphs[r];
  auto sig = graph_signature(c);
  sig.push_back((uintptr_t)c->red.p);
  sig.push_back((uintptr_t)c->scal.p);
  sig.push_back((uintptr_t)c->flags.p);
  if (!(g.exec && g.sig == sig)) {
    destroy_graph(g);
    g.sig = sig;
    if (!c->cap_stream) XM_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    // first use: run it eagerly (allocations / plans happen outside any capture)
    post_tcg_sequence(c, r);
    sync(c);
    cudaStream_t orig = c->stream;
    const int64_t l0 = c->stats.kernel_launches, s0 = c->stats.spmm_calls;
    c->stream = c->cap_stream;
    cudaGraph_t graph = nullptr;
    bool ok = true;
    try {
      XM_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
      post_tcg_sequence(c, r);
      XM_CUDA(cudaStreamEndCapture(c->cap_stream, &graph));
    } catch (...) {
      cudaStreamEndCapture(c->cap_stream, &graph);
      cudaGetLastError();
      ok = false;
    }
    c->stream = orig;
    g.launches = c->stats.kernel_launches - l0;
    g.spmms = c->stats.spmm_calls - s0;
    c->stats.kernel_launches = l0;
    c->stats.spmm_calls = s0;
    if (ok && cudaGraphInstantiate(&g.exec, graph, 0) != cudaSuccess) {
      cudaGetLastError();
      g.exec = nullptr;
    }
    if (graph) cudaGraphDestroy(graph);
    return;  // this iteration's step already ran eagerly (and was counted)
  }
  XM_CUDA(cudaGraphLaunch(g.exec, c->stream));
  c->stats.kernel_launches += g.launches;
  c->stats.spmm_calls += g.spmms;
}

struct RtrOut {
  bool converged = false;
  int64_t outer = 0;
  double f = 0, g2 = 0, amin = 0;
};

// Riemannian trust region with device-state tCG (O5).
RtrOut rtr(xm_ctx* c, double tol_abs) {
  const int r = c->r;
  const int64_t len = (int64_t)c->n * r;
  const xm_options& o = c->opt;
  const double Delta0 = o.delta0_coef * std::sqrt(3.0 * c->N);
  const double Dbar = o.delta_max_mult * Delta0;
  double Delta = Delta0;
  RtrOut out;
  double f, g2, amin;
  PhaseClock pc(c);
  eval_point(c, &f, &g2, &amin);
  pc.lap(3);
  int64_t accepts = 0;
  int64_t it = 0;
  const double eps = 2.220446049250313e-16;
  for (it = 0;; ++it) {
    if (std::sqrt(g2) <= tol_abs) {
      out.converged = true;
      break;
    }
    if (it >= o.max_outer) break;
    // ---- tCG (device-resident state; persistent / fused / three-kernel)
    bool deferred = false;
    TcgState hs = run_tcg(c, r, Delta, c->phases_on ? nullptr : &deferred);
    if (!deferred) c->info.hvps += hs.n_hvp;
    pc.lap(0);
    // ---- retraction (+ ⟨g,η⟩, ⟨η,Hη⟩) and cancellation-free Δf (reading C21)
    post_tcg(c, r);
    // one host round trip: Δf terms, the App. D term, the retraction flag and
    // (deferred) the tCG state, all through the pinned host scalars
    double* hp = c->hpin;
    XM_CUDA(cudaMemcpyAsync(hp + kPinD, c->scal.p + 8, 4 * 8, cudaMemcpyDeviceToHost, c->stream));
    if (o.scale_reg != 0.0)
      XM_CUDA(cudaMemcpyAsync(hp + kPinD + 4, c->scal.p + 26, 8, cudaMemcpyDeviceToHost, c->stream));
    XM_CUDA(cudaMemcpyAsync(hp + kPinD + 5, c->flags.p, 4, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (deferred) {
      hs = tcg_deferred_state(c);
      c->info.hvps += hs.n_hvp;
    }
    const double d[4] = {hp[kPinD], hp[kPinD + 1], hp[kPinD + 2], hp[kPinD + 3]};
    const double dreg = (o.scale_reg != 0.0) ? hp[kPinD + 4] : 0.0;
    int rerr = 0;
    std::memcpy(&rerr, hp + kPinD + 5, 4);
    if (rerr) throw Error(XM_ERETRACT, "retraction failure");
    pc.lap(1);
    const double df = 2.0 * d[0] + d[1] + dreg;
    const double model_dec = -d[2] - 0.5 * d[3];
    const double reg = std::max(1.0, std::fabs(f)) * eps * 1e3;
    const double rho = (-df + reg) / (model_dec + reg);
    const bool limited = (hs.stop == TCG_NEGCURV || hs.stop == TCG_EXCEEDED);
    if (!(rho >= 0.25) || std::isnan(rho)) Delta /= 4.0;
    else if (rho > 0.75 && limited) Delta = std::min(2.0 * Delta, Dbar);
    if (rho > o.rho_prime) {
      XM_CUDA(cudaMemcpyAsync(c->Y.p, c->Ynew.p, len * 8, cudaMemcpyDeviceToDevice, c->stream));
      ++accepts;
      if (o.refresh_every > 0 && accepts % o.refresh_every == 0) {
        grad_fused(c, r, c->Y.p, c->QY.p, c->grad.p, c->scal.p);
      } else {
        axpy(c, len, 1.0, c->QD.p, c->QY.p);
        grad_and_multipliers(c, r, c->Y.p, c->QY.p, c->grad.p, c->scal.p);
      }
      double h[3];
      read_scal(c, 0, 3, h);
      f = h[0];
      g2 = h[1];
      amin = h[2];
    }
    pc.lap(2);
  }
  // fresh Q·Y before any certificate (O4)
  eval_point(c, &f, &g2, &amin);
  pc.lap(3);
  out.outer = it;
  out.f = f;
  out.g2 = g2;
  out.amin = amin;
  c->info.outer_iters += it;
  return out;
}

// Certificate at the current point (Alg. 1 lines 9-12): Λ from the last gradient
// pass; λ_min(Z) by Lanczos on Z.  If Lanczos has not converged within ≈ the
// cost of one dense factorisation (n/72 steps) — the clustered small end of
// Z's spectrum on banded scenes — Z ⪰ −εI is decided by Cholesky of Z + εI
// (single GPU), and λ_min is then computed by shift-invert Lanczos on
// (Z + εI)⁻¹ = L⁻ᵀL⁻¹ (X = L⁻¹ by the DMMA TRSM; a handful of steps: the
// inverted spectrum is well separated).  A second Cholesky at a small shift δ
// (just above max(0, −λ_min) and the backward-error floor) then proves the
// tight lower bound λ_min ≥ −δ − γ·tr(Z+δI) − u‖Z‖_F (lower_rigorous).  Only
// if Z + εI is not PD does Lanczos on Z continue to convergence (the escape
// needs v).
void certify_current(xm_ctx* c, double* lambda, int* steps) {
  const double tol = c->opt.eig_tol * std::max(1.0, c->normQ);
  const double eps = c->opt.cert_tol * std::max(1.0, c->normQ);
  c->cert_method = 0;
  c->cert_rigorous = 0;
  if (c->opt.scale_reg != 0.0) reg_frames(c, c->r, c->Y.p, nullptr, c->scal.p + 24);  // d_i at Y
  if (dense_fused(c) && c->opt.cert_cholesky) {
    int budget = std::min(c->opt.lanczos_max, std::max(32, c->n / 72));
    PhaseClock pc(c);
    bool conv;
    {
      NvtxRange r_("lanczos(Z)");
      conv = lanczos(c, tol, budget, lambda, steps, c->cert_v.p);
    }
    pc.lap(6);
    double low_eps = 0.0;
    DBuf<double>& U = scratch_f64(c, "zw_U");
    if (conv) {
      c->cert_lower = *lambda;
    } else if (U.alloc((size_t)c->n * c->ldq),
               psd_test_cholesky(c, eps, &low_eps, U.p, c->ldq) && (pc.lap(7), true)) {
      c->cert_method = 1;
      c->cert_lower = low_eps;
      c->cert_rigorous = 1;
      DBuf<double>& X = scratch_f64(c, "zw_X");
      X.alloc((size_t)c->n * c->ldq);
      identity(c, X.p, c->n, c->ldq);
      dense_trsm_lower_left(c, c->Zw.p, c->n, c->ldq, U.p, c->ldq, X.p, c->n, c->ldq, true);
      double th = 0.0;
      int s2 = 0;
      LanczosOp op;
      op.X = X.p;
      op.ldx = c->ldq;
      lanczos(c, tol, c->opt.lanczos_max, &th, &s2, c->cert_v.p, op);
      *steps += s2;
      *lambda = (th < 0.0) ? -1.0 / th - eps : -eps;
      pc.lap(6);
      // tight proven bound: Cholesky at δ just above max(0, −λ_min) and the backward-error floor
      const double floor_b = -(low_eps + eps);
      const double delta = std::max(8.0 * floor_b, 2.0 * std::max(0.0, -*lambda));
      double low_d = 0.0;
      if (delta < eps && psd_test_cholesky(c, delta, &low_d)) c->cert_lower = low_d;
      pc.lap(7);
    } else {
      int s1 = *steps;
      lanczos(c, tol, c->opt.lanczos_max, lambda, steps, c->cert_v.p);
      *steps += s1;
      c->cert_lower = *lambda;
    }
  } else {
    lanczos(c, tol, c->opt.lanczos_max, lambda, steps, c->cert_v.p);
    c->cert_lower = *lambda;
  }
  c->cert_valid = true;
  c->cert_lambda = *lambda;
  c->cert_steps = *steps;
  c->info.lanczos_steps += *steps;
}

// Escape along D = [0, v] from [Y, 0] (Thm 2, Alg. 1 l.14-22, reading C9)
void escape(xm_ctx* c) {
  const int r = c->r;
  const int r1 = r + 1;
  const int64_t len1 = (int64_t)c->n * r1;
  pad_column(c, r, c->Y.p, c->Ynew.p, c->cert_v.p, c->dir.p);   // Yz, Dz
  pad_column(c, r, c->QY.p, c->Heta.p, nullptr, nullptr);       // QYz
  double alpha = 1.0;
  for (int h = 0; h <= 60; ++h) {
    XM_CUDA(cudaMemsetAsync(c->flags.p, 0, sizeof(int), c->stream));
    retract(c, r1, c->Ynew.p, c->dir.p, alpha, c->eta.p, c->Dv.p, c->flags.p);
    df_product(c, r1, c->Dv.p, c->Heta.p, c->QD.p, c->scal.p + 8);
    double d[2];
    read_scal(c, 8, 2, d);
    double dreg = 0.0;
    if (c->opt.scale_reg != 0.0) {
      reg_frames(c, r1, c->Ynew.p, c->Dv.p, c->scal.p + 24);
      read_scal(c, 26, 1, &dreg);
    }
    double df = 2.0 * d[0] + d[1] + dreg;
    if (df < 0.0) {
      XM_CUDA(cudaMemcpyAsync(c->Y.p, c->eta.p, len1 * 8, cudaMemcpyDeviceToDevice, c->stream));
      c->r = r1;
      c->info.escapes++;
      return;
    }
    alpha *= 0.5;
  }
  throw Error(XM_EESCAPE, "escape failed");
}

__global__ void k_identity_init(int N, int r, double* Y) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)3 * N * r) return;
  int64_t row = t / r;
  int col = (int)(t % r);
  Y[t] = (col == (int)(row % 3)) ? 1.0 : 0.0;
}

void destroy_graphs(xm_ctx* c) {
  for (auto& g : c->tcg_graphs) destroy_graph(g);
  for (auto& g : c->post_graphs) destroy_graph(g);
}

void reset_after_new_Q(xm_ctx* c) {
  c->stage = 1;
  c->factor_set = false;
  c->cert_valid = false;
  c->have_round = false;
  c->r = 0;
  alloc_vectors(c);
}

}  // namespace

// =============================================================================
extern "C" {

void xm_default_options(xm_options* o) {
  if (!o) return;
  o->grad_tol = 1e-10;
  o->delta0_coef = 0.1;
  o->delta_max_mult = 10.0;
  o->rho_prime = 0.1;
  o->tcg_kappa = 0.1;
  o->tcg_theta = 1.0;
  o->eig_tol = 1e-8;
  o->cert_tol = 1e-6;
  o->scale_floor = 1e-3;
  o->tcg_max_inner = 500;
  o->max_outer = 5000;
  o->rank_cap = 10;
  o->lanczos_max = 3000;
  o->refresh_every = 50;
  o->profile = 0;
  o->cert_cholesky = 1;
  o->spmm_kernel = 0;
  o->seed = 0;
  o->scale_reg = 0.0;
  o->implicit_q = -1;  // auto: matrix-free where its modelled product time is smaller
}

const char* xm_strerror(xm_status s) {
  switch (s) {
    case XM_OK: return "ok (certified)";
    case XM_UNCERTIFIED: return "uncertified: rank cap reached with lambda_min(Z) < -cert_tol";
    case XM_NOT_CONVERGED: return "trust region did not converge";
    case XM_EINVAL: return "invalid argument";
    case XM_EDISCONNECTED: return "graph numerically disconnected";
    case XM_ENOMEM: return "out of device memory";
    case XM_ECUDA: return "CUDA error";
    case XM_ENCCL: return "NCCL error";
    case XM_ERETRACT: return "retraction failure";
    case XM_EESCAPE: return "escape failed";
    case XM_EINFEASIBLE: return "infeasible point";
    case XM_EDEGENERATE: return "degenerate block";
    case XM_ESTATE: return "call order violated";
  }
  return "unknown status";
}

xm_status xm_shard_rows(int32_t N, int32_t world, int32_t rank, int32_t* f0, int32_t* f1,
                        int32_t* frames_per_rank) {
  if (N < 1 || world < 1 || rank < 0 || rank >= world || !f0 || !f1) return XM_EINVAL;
  int a, b, nfpr;
  shard_of(N, world, rank, &a, &b, &nfpr);
  *f0 = a;
  *f1 = b;
  if (frames_per_rank) *frames_per_rank = nfpr;
  return XM_OK;
}

xm_status xm_nccl_unique_id(void* out128) {
  if (!out128) return XM_EINVAL;
  try {
    nccl_unique_id(out128);
    return XM_OK;
  } catch (const Error& e) {
    return e.code;
  }
}

xm_status xm_create(xm_ctx** out, int device, int rank, int world, const void* nccl_id,
                    const xm_options* opts, void* cuda_stream) {
  if (!out || world < 1 || rank < 0 || rank >= world) return XM_EINVAL;
  *out = nullptr;
  xm_ctx* c = new xm_ctx();
  c->device = device;
  c->rank = rank;
  c->world = world;
  if (opts) c->opt = *opts; else xm_default_options(&c->opt);
  // A/B switches for measurements (the defaults are the production path)
  if (std::getenv("XM_NO_SYM")) c->opt.spmm_kernel = 1;
  if (std::getenv("XM_FORCE_SYM")) c->opt.spmm_kernel = 2;
  if (std::getenv("XM_PHASES")) c->phases_on = true;
  if (std::getenv("XM_NO_FUSED_TCG")) c->fused_tcg = false;
  if (std::getenv("XM_NO_PERSIST_TCG")) c->persist_tcg = false;
  if (const char* e = std::getenv("XM_GEMM_TILE"))
    c->gemm_tile = std::string(e) == "bk16" ? 1 : std::string(e) == "mid" ? 2 : std::string(e) == "w8" ? 3 : 0;
  if (const char* e = std::getenv("XM_TRSM_SB")) c->trsm_sb = std::max(64, atoi(e) / 64 * 64);
  if (std::getenv("XM_SYM_TCG")) c->persist_sym = 1;
  if (std::getenv("XM_NO_SYM_TCG")) c->persist_sym = -1;
  if (std::getenv("XM_NO_GRAPHS")) c->use_graphs = false;
  if (c->opt.rank_cap > XM_MAX_R) c->opt.rank_cap = XM_MAX_R;
  xm_status st = guard(c, [&] {
    if (cuda_stream) {
      c->stream = (cudaStream_t)cuda_stream;
    } else {
      XM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    XM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->hpin), kPinDoubles * sizeof(double)));
    nccl_init(c, nccl_id);
  });
  if (st != XM_OK) {
    xm_destroy(c);
    return st;
  }
  *out = c;
  return XM_OK;
}

void xm_destroy(xm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_persist)
    if (e) cudaEventDestroy(e);
  destroy_graphs(c);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  if (c->hpin) cudaFreeHost(c->hpin);
  for (int q = 0; q < xm_ctx::kTrsmStreams; ++q)
    if (c->trsm_streams[q]) cudaStreamDestroy(c->trsm_streams[q]);
  for (int q = 0; q <= xm_ctx::kTrsmStreams; ++q)
    if (c->trsm_ev[q]) cudaEventDestroy(c->trsm_ev[q]);
  if (c->ev_la) cudaEventDestroy(c->ev_la);
  if (c->ev_lb) cudaEventDestroy(c->ev_lb);
  nccl_destroy(c);
  sym_plan_destroy(c);
  sym_plan_slot_destroy(c->imp_sym_plan);
  sym_tcg_plan_destroy(c);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

xm_status xm_build_Q(xm_ctx* c, int32_t N, int32_t M, int64_t E, const int32_t* frame,
                     const int32_t* landmark, const double* lifted_pts, const double* weights) {
  if (!c) return XM_EINVAL;
  if (!frame || !landmark || !lifted_pts) return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_build_Q");
    double t0 = now_ms();
    c->stage = 0;
    c->orig_in.release();  // the caller's input order
    build_Q_device(c, N, M, E, frame, landmark, lifted_pts, weights);
    c->E_user = E;
    reset_after_new_Q(c);
    sync(c);
    c->stats.ms_build += now_ms() - t0;
  });
}

__global__ void k_copy_rows(int rows, int n, const double* __restrict__ src, int64_t lds,
                            double* __restrict__ dst, int64_t ldd) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)rows * n) return;
  int i = (int)(t / n), j = (int)(t % n);
  dst[(int64_t)i * ldd + j] = src[(int64_t)i * lds + j];
}

xm_status xm_set_Q(xm_ctx* c, int32_t N, const double* Q_full) {
  if (!c || N < 1 || !Q_full) return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_set_Q");
    c->implicit_active = false;  // a dense Q from the caller
    c->N = N;
    c->M = 0;
    c->E = 0;
    c->n = 3 * N;
    c->ldq = round_up(c->n, 32);
    c->ldk = round_up(std::max(N - 1, 1), 32);
    set_shard(c, N);
    c->Q.alloc((size_t)std::max(c->nrows, 1) * c->ldq);
    const int64_t n = c->n;
    if (c->nrows > 0) {
      XM_CUDA(cudaMemcpy2DAsync(c->Q.p, c->ldq * 8, Q_full + (int64_t)c->row0 * n, n * 8, n * 8,
                                c->nrows,
                                is_device_ptr(Q_full) ? cudaMemcpyDeviceToDevice
                                                      : cudaMemcpyHostToDevice,
                                c->stream));
    }
    c->have_recovery = false;
    c->nnzb = 0;
    // ‖Q‖_F
    DBuf<double> part;
    part.alloc(kDotBlocks);
    DBuf<double> tmp;
    tmp.alloc((size_t)std::max(c->nrows, 1) * n);
    k_copy_rows<<<ceil_div((int64_t)c->nrows * n, 256), 256, 0, c->stream>>>(c->nrows, (int)n, c->Q.p,
                                                                           c->ldq, tmp.p, n);
    dot_flat(c, tmp.p, tmp.p, (int64_t)c->nrows * n, part.p, kDotBlocks);
    c->scal.alloc(64);
    reduce_partials(c, part.p, kDotBlocks, 1, c->scal.p);
    if (c->world > 1) nccl_allreduce_sum(c, c->scal.p, 1);
    double s2 = 0;
    XM_CUDA(cudaMemcpyAsync(&s2, c->scal.p, 8, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    c->normQ = std::sqrt(s2);
    c->stats.q_bytes = (int64_t)c->nrows * n * 8;
    reset_after_new_Q(c);
  });
}

xm_status xm_solve(xm_ctx* c, int32_t r0, double tol, xm_solve_info* info) {
  if (!c) return XM_EINVAL;
  xm_status result = XM_OK;
  xm_status st = guard(c, [&] {
    NvtxRange nvtx_("xm_solve");
    require_stage(c, 1);
    double t0 = now_ms();
    c->info = xm_solve_info{};
    if (!c->factor_set) {
      if (r0 < 3 || r0 > XM_MAX_R) throw Error(XM_EINVAL, "r0 must be in [3, 12]");
      c->r = r0;
      int64_t len = (int64_t)c->n * r0;
      k_identity_init<<<ceil_div(len, 256), 256, 0, c->stream>>>(c->N, r0, c->Y.p);
      XM_CHECK_LAUNCH();
      count_launch(c);
    }
    c->factor_set = false;
    const double tol_abs = (tol > 0 ? tol : c->opt.grad_tol) * std::max(1.0, c->normQ);
    const int64_t spmm0 = c->stats.spmm_calls;
    bool certified = false;
    RtrOut ro;
    double lam = 0.0;
    while (true) {
      ro = rtr(c, tol_abs);
      int steps = 0;
      PhaseClock pc(c);
      certify_current(c, &lam, &steps);
      pc.lap(4);
      certified = ro.converged && c->cert_lower >= -c->opt.cert_tol * std::max(1.0, c->normQ);
      if (certified || !ro.converged || c->r >= c->opt.rank_cap) break;
      escape(c);
      pc.lap(5);
    }
    if (c->phases_on) {
      for (int k = 0; k < 8; ++k)
        if (c->phase_n[k])
          fprintf(stderr, "[xm phases] %-12s %9.3f ms  (%lld laps)\n", kPhaseNames[k], c->phase_ms[k],
                  c->phase_n[k]);
      for (int k = 0; k < 8; ++k) c->phase_ms[k] = 0.0, c->phase_n[k] = 0;
      if (c->tdbg.p) {  // stamps of the last fused tCG iteration that ran to its end
        std::vector<unsigned long long> h(148 * 8);
        XM_CUDA(cudaMemcpy(h.data(), c->tdbg.p, h.size() * 8, cudaMemcpyDeviceToHost));
        const int G = std::min(148, c->N);
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < G; ++b) t0 = std::min(t0, h[b * 8]);
        const char* nm[8] = {"start", "loop end", "pre-bar1", "post-bar1", "pre-bar2", "post-bar2",
                             "end", "assembled"};  // persistent kernel: stamps of iteration 1
        for (int k = 0; k < 8; ++k) {
          std::vector<double> v;
          for (int b = 0; b < G; ++b)
            if (h[b * 8 + k]) v.push_back((h[b * 8 + k] - t0) * 1e-3);
          if (v.empty()) continue;
          std::sort(v.begin(), v.end());
          fprintf(stderr, "[xm fused tCG] %-9s min %7.2f  med %7.2f  max %7.2f us\n", nm[k], v.front(),
                  v[v.size() / 2], v.back());
        }
        if (std::getenv("XM_PHASES_CTA")) {  // per-CTA stream end (stamp 1), for balance studies
          fprintf(stderr, "[xm fused tCG] loop end per CTA:");
          for (int b = 0; b < G; ++b) fprintf(stderr, " %.1f", (h[b * 8 + 1] - t0) * 1e-3);
          fprintf(stderr, "\n[xm fused tCG] assembly per CTA:");
          for (int b = 0; b < G; ++b) fprintf(stderr, " %.1f", (h[b * 8 + 7] - h[b * 8 + 3]) * 1e-3);
          fprintf(stderr, "\n[xm fused tCG] camera per CTA:");
          for (int b = 0; b < G; ++b) fprintf(stderr, " %.1f", (h[b * 8 + 4] - h[b * 8 + 7]) * 1e-3);
          fprintf(stderr, "\n");
        }
      }
    }
    c->info.f = ro.f;
    c->info.grad_norm = std::sqrt(ro.g2);
    c->info.lambda_min = lam;
    c->info.normQ = c->normQ;
    c->info.s_min = c->N > 1 ? std::sqrt(std::max(ro.amin, 0.0)) : 1.0;
    c->info.r = c->r;
    c->info.certified = certified;
    c->info.converged = ro.converged;
    c->info.spmms = c->stats.spmm_calls - spmm0;
    c->stage = 2;
    c->have_round = false;
    c->stats.ms_solve += now_ms() - t0;
    if (!ro.converged) result = XM_NOT_CONVERGED;
    else if (!certified) result = XM_UNCERTIFIED;
    if (c->N > 1 && c->info.s_min < 1e-8) throw Error(XM_EDEGENERATE, "scale collapse s_i < 1e-8");
  });
  if (info && c) *info = c->info;
  return st != XM_OK ? st : result;
}

xm_status xm_certify(xm_ctx* c, xm_certificate* out, double* min_eigvec) {
  if (!c) return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_certify");
    require_stage(c, 1);
    if (c->r == 0) throw Error(XM_ESTATE, "no factor: call xm_solve or xm_set_factor first");
    double t0 = now_ms();
    double f, g2, amin;
    eval_point(c, &f, &g2, &amin);
    double lam;
    int steps;
    if (c->cert_valid) {
      lam = c->cert_lambda;
      steps = c->cert_steps;
    } else {
      certify_current(c, &lam, &steps);
    }
    round_recover_device(c);
    // ρ̂ = f(Ŷ) at the rounded factor
    spmm_full(c, c->Yr.p, 3, c->tmp.p, nullptr);
    const double* A[2] = {c->Yr.p, c->Y.p};
    const double* B[2] = {c->tmp.p, c->Y.p};
    double d[2];
    dots(c, (int64_t)c->n * 3, 1, A, B, d);
    double trX;
    {
      const double* A2[1] = {c->Y.p};
      const double* B2[1] = {c->Y.p};
      dots(c, (int64_t)c->n * c->r, 1, A2, B2, &trX);
    }
    double l0[3];
    XM_CUDA(cudaMemcpyAsync(l0, c->lam.p, 24, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    double reg_dual = 0.0, reg_hat = 0.0;
    if (c->opt.scale_reg != 0.0) {  // App. D: ρ_dual −= λΣ(α²−1) at Y; ρ̂ += F(Ŷ)
      double t[3];
      reg_frames(c, 3, c->Yr.p, nullptr, c->scal.p + 24);
      read_scal(c, 24, 1, &reg_hat);
      reg_frames(c, c->r, c->Y.p, nullptr, c->scal.p + 24);  // leaves d_i at Y in c->regd
      read_scal(c, 24, 3, t);
      reg_dual = -c->opt.scale_reg * t[1];
    }
    xm_certificate ce{};
    ce.lambda_min = lam;
    ce.lambda_lower = c->cert_lower;
    ce.method = c->cert_method;
    ce.rho_dual = l0[0] + l0[1] + l0[2] + reg_dual;
    ce.rho_hat = d[0] + reg_hat;
    ce.trace_X = trX;
    // η (Eq. (13)) with ρ_SDP bounded below by ρ_dual + min(0, λ)·tr X̂ (reading
    // C10): once with the converged λ_min (estimate), once with the proven λ_lower
    auto eta_of = [&](double lo) {
      return (ce.rho_hat - lo) / (1.0 + std::fabs(ce.rho_hat) + std::fabs(lo));
    };
    ce.rho_lower = ce.rho_dual + std::min(0.0, lam) * trX;
    ce.eta = eta_of(ce.rho_lower);
    ce.rho_lower_rigorous = ce.rho_dual + std::min(0.0, c->cert_lower) * trX;
    ce.eta_rigorous = eta_of(ce.rho_lower_rigorous);
    ce.lower_rigorous = c->cert_rigorous;
    double lowE = std::max(0.0, lam) * trX + ce.rho_dual;
    ce.eta_E = eta_of(lowE);
    ce.kkt_resid = 0.5 * std::sqrt(g2);  // grad = 2 Z Y
    ce.grad_norm = std::sqrt(g2);
    ce.normQ = c->normQ;
    ce.lanczos_steps = steps;
    ce.certified = (std::min(lam, c->cert_lower) >= -c->opt.cert_tol * std::max(1.0, c->normQ)) &&
                   std::sqrt(g2) <= c->opt.grad_tol * std::max(1.0, c->normQ) * 1.0001;
    c->cert = ce;
    c->have_cert = true;
    if (out) *out = ce;
    if (min_eigvec) copy_out(c, min_eigvec, c->cert_v.p, (size_t)c->n * 8);
    c->stats.ms_certify += now_ms() - t0;
  });
}

xm_status xm_round_recover(xm_ctx* c, double* R, double* s, double* t, double* p,
                           int32_t* n_flipped) {
  if (!c) return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_round_recover");
    require_stage(c, 1);
    if (c->r == 0) throw Error(XM_ESTATE, "no factor");
    double t0 = now_ms();
    if (!c->have_round) round_recover_device(c);
    copy_out(c, R, c->Rs.p, (size_t)c->N * 9 * 8);
    copy_out(c, s, c->s_out.p, (size_t)c->N * 8);
    copy_out(c, t, c->t_out.p, (size_t)c->N * 3 * 8);
    if (p && c->M > 0) copy_out(c, p, c->p_out.p, (size_t)c->M * 3 * 8);
    if (n_flipped) *n_flipped = c->n_flipped;
    sync(c);
    c->stats.ms_round += now_ms() - t0;
  });
}

// ----------------------------------------------------------------- XM²
// SURVEY §8(f) NEXT-2 (reading C22): residuals
// of the measurements at the recovered solution, and the drop-10%-and-rebuild
// step (the caller then solves / certifies / rounds again).
xm_status xm_edge_residuals(xm_ctx* c, double* res) {
  if (!c || !res) return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_edge_residuals");
    require_stage(c, 1);
    if (c->r == 0) throw Error(XM_ESTATE, "no factor");
    if (!c->have_recovery) throw Error(XM_ESTATE, "no view graph (Q was set directly)");
    if (!c->have_round) round_recover_device(c);
    DBuf<double>& out = scratch_f64(c, "xm2_user_res");
    out.alloc(std::max<int64_t>(c->E_user, 1));
    edge_residuals_user(c, out.p);
    copy_out(c, res, out.p, (size_t)c->E_user * 8);
    sync(c);
  });
}

xm_status xm_xm2(xm_ctx* c, double drop_fraction, uint8_t* keep, int64_t* n_dropped, int64_t* n_restored) {
  if (!c || !(drop_fraction >= 0.0 && drop_fraction < 1.0)) return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_xm2");
    require_stage(c, 1);
    if (c->r == 0) throw Error(XM_ESTATE, "no factor");
    if (!c->have_recovery) throw Error(XM_ESTATE, "no view graph (Q was set directly)");
    const double t0 = now_ms();
    if (!c->have_round) round_recover_device(c);
    DBuf<uint32_t>& kb = scratch_u32(c, "xm2_user_keep");
    kb.alloc((size_t)c->E_user / 4 + 2);
    uint8_t* kd = reinterpret_cast<uint8_t*>(kb.p);
    try {
      xm2_device(c, drop_fraction, kd, n_dropped, n_restored);
    } catch (...) {
      // the measurement mapping / canonical arrays may be half-rebuilt: no Q
      // to solve on until the next xm_build_Q (xm.h: a failed call must not
      // leave a context whose stage and data disagree)
      c->stage = 0;
      c->have_recovery = false;
      throw;
    }
    reset_after_new_Q(c);
    if (keep) copy_out(c, keep, kd, (size_t)c->E_user);
    sync(c);
    c->stats.ms_build += now_ms() - t0;
  });
}

// ----------------------------------------------------------------- hooks
xm_status xm_get_S_pattern(xm_ctx* c, int64_t* rowptr, int32_t* colidx, int64_t* nnzb) {
  if (!c) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    if (!c->have_recovery) throw Error(XM_ESTATE, "no view graph (Q was set directly)");
    if (!c->pattern_valid) build_s_pattern(c, c->N);  // matrix-free builds: on demand
    if (nnzb) *nnzb = c->nnzb;
    if (rowptr) copy_out(c, rowptr, c->s_rowptr.p, (size_t)(c->N + 1) * 8);
    if (colidx) copy_out(c, colidx, c->s_colidx.p, (size_t)c->nnzb * 4);
    sync(c);
  });
}

xm_status xm_get_Q_rows(xm_ctx* c, int32_t row0, int32_t nrows, double* out) {
  if (!c || !out) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    if (c->implicit_active) throw Error(XM_EINVAL, "Q is not formed in the implicit (NEXT-1) mode");
    if (row0 < c->row0 || row0 + nrows > c->row0 + c->nrows || nrows < 0)
      throw Error(XM_EINVAL, "rows not owned by this rank");
    if (nrows == 0) return;
    XM_CUDA(cudaMemcpy2DAsync(out, (size_t)c->n * 8, c->Q.p + (int64_t)(row0 - c->row0) * c->ldq,
                              c->ldq * 8, (size_t)c->n * 8, nrows,
                              is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                              c->stream));
    sync(c);
    if (c->world > 1 && c->have_recovery && !is_device_ptr(out)) {
      // band layout: only the lower trapezoid (columns ≤ row) is this rank's data
      for (int32_t i = 0; i < nrows; ++i)
        for (int64_t j = row0 + i + 1; j < c->n; ++j) out[(int64_t)i * c->n + j] = NAN;
    }
  });
}

xm_status xm_spmm(xm_ctx* c, const double* V, double* out, int32_t r) {
  if (!c || !V || !out || r < 1 || r > XM_MAX_R) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    int64_t len = (int64_t)c->n * r;
    copy_in(c, c->hV.p, V, len * 8);
    spmm_full(c, c->hV.p, r, c->hO.p, nullptr);
    copy_out(c, out, c->hO.p, len * 8);
    sync(c);
  });
}

xm_status xm_grad(xm_ctx* c, const double* Y, double* grad, double* f, int32_t r) {
  if (!c || !Y || r < 1 || r > XM_MAX_R) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    int64_t len = (int64_t)c->n * r;
    copy_in(c, c->hY.p, Y, len * 8);
    grad_fused(c, r, c->hY.p, c->hQY.p, c->hO.p, c->scal.p + 20);
    if (grad) copy_out(c, grad, c->hO.p, len * 8);
    if (f) read_scal(c, 20, 1, f);
    sync(c);
    c->cert_valid = false;  // Λ buffer now holds the hook's multipliers
  });
}

xm_status xm_hvp(xm_ctx* c, const double* Y, const double* V, double* HV, int32_t r) {
  if (!c || !Y || !V || !HV || r < 1 || r > XM_MAX_R) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    int64_t len = (int64_t)c->n * r;
    copy_in(c, c->hY.p, Y, len * 8);
    copy_in(c, c->hV.p, V, len * 8);
    grad_fused(c, r, c->hY.p, c->hQY.p, c->hO.p, c->scal.p + 20);
    c->part1.alloc(2048);
    hvp_product(c, r, c->hY.p, c->hV.p, c->hO.p, c->part1.p, nullptr);
    copy_out(c, HV, c->hO.p, len * 8);
    sync(c);
    c->cert_valid = false;
  });
}

xm_status xm_tcg(xm_ctx* c, const double* Y, int32_t r, double Delta, int32_t path, double* eta,
                 double* Heta, int32_t* n_hvp, int32_t* stop) {
  if (!c || !Y || !eta || r < 1 || r > XM_MAX_R || !(Delta > 0.0) || path < 0 || path > 4)
    return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_tcg");
    require_stage(c, 1);
    const bool f0 = c->fused_tcg, p0 = c->persist_tcg;
    const int s0 = c->persist_sym;
    struct Restore {
      xm_ctx* c; bool f, p; int s;
      ~Restore() { c->fused_tcg = f; c->persist_tcg = p; c->persist_sym = s; }
    } restore{c, f0, p0, s0};
    switch (path) {
      case 1: c->fused_tcg = c->persist_tcg = true; c->persist_sym = 1; break;
      case 2: c->fused_tcg = c->persist_tcg = true; c->persist_sym = -1; break;
      case 3: c->fused_tcg = true; c->persist_tcg = false; break;
      case 4: c->fused_tcg = false; break;
      default: break;
    }
    const bool ok = path == 0 ||
                    (path == 1 && tcg_persist_sym_supported(c, r)) ||
                    (path == 2 && !tcg_persist_sym_supported(c, r) && tcg_persist_supported(c, r)) ||
                    (path == 3 && !tcg_persist_supported(c, r) && tcg_fused_supported(c, r)) ||
                    (path == 4 && !tcg_persist_supported(c, r));
    if (!ok) throw Error(XM_EINVAL, "tCG path not available for this problem / rank");
    const int64_t len = (int64_t)c->n * r;
    c->r = r;
    copy_in(c, c->Y.p, Y, len * 8);
    c->factor_set = true;
    c->cert_valid = false;
    c->have_round = false;
    grad_fused(c, r, c->Y.p, c->QY.p, c->grad.p, c->scal.p);   // g, Λ, ‖g‖² (scal[1])
    const TcgState hs = run_tcg(c, r, Delta);
    copy_out(c, eta, c->eta.p, len * 8);
    if (Heta) copy_out(c, Heta, c->Heta.p, len * 8);
    sync(c);
    if (n_hvp) *n_hvp = hs.n_hvp;
    if (stop) *stop = hs.stop;
  });
}

xm_status xm_solve_batch(xm_ctx* c, int32_t B, int32_t N, const double* Q, int64_t q_stride,
                         const double* Y0, int32_t r0, double* Y_out, xm_batch_result* res) {
  if (!c || B < 1 || N < 1 || !Q || !Y0 || !Y_out || !res || q_stride < 0) return XM_EINVAL;
  return guard(c, [&] {
    NvtxRange nvtx_("xm_solve_batch");
    const int64_t n = 3 * (int64_t)N;
    const int64_t qcount = q_stride == 0 ? n * n : (B - 1) * q_stride + n * n;
    const double* Qd = Q;
    const double* Yd = Y0;
    DBuf<double>& qb = scratch_f64(c, "batch_q");
    DBuf<double>& yb = scratch_f64(c, "batch_y0");
    DBuf<double>& yo = scratch_f64(c, "batch_yout");
    DBuf<uint64_t>& rb = scratch_u64(c, "batch_res");
    if (!is_device_ptr(Q)) {
      qb.alloc((size_t)qcount);
      copy_in(c, qb.p, Q, (size_t)qcount * 8);
      Qd = qb.p;
    }
    if (!is_device_ptr(Y0)) {
      yb.alloc((size_t)B * n * r0);
      copy_in(c, yb.p, Y0, (size_t)B * n * r0 * 8);
      Yd = yb.p;
    }
    const bool dev_out = is_device_ptr(Y_out);
    double* Yo = Y_out;
    if (!dev_out) {
      yo.alloc((size_t)B * n * 8);
      Yo = yo.p;
    }
    rb.alloc((sizeof(xm_batch_result) * (size_t)B + 7) / 8);
    xm_batch_result* rd = reinterpret_cast<xm_batch_result*>(rb.p);
    batch_staircase(c, B, N, Qd, q_stride, Yd, r0, Yo, rd);
    if (!dev_out) copy_out(c, Y_out, Yo, (size_t)B * n * 8 * 8);
    copy_out(c, res, rd, sizeof(xm_batch_result) * (size_t)B);
    sync(c);
  });
}

xm_status xm_project(xm_ctx* c, const double* Y, const double* W, double* out, int32_t r) {
  if (!c || !Y || !W || !out || r < 1 || r > XM_MAX_R) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    int64_t len = (int64_t)c->n * r;
    copy_in(c, c->hY.p, Y, len * 8);
    copy_in(c, c->hV.p, W, len * 8);
    project(c, r, c->hY.p, c->hV.p, c->hO.p);
    copy_out(c, out, c->hO.p, len * 8);
    sync(c);
  });
}

xm_status xm_retract(xm_ctx* c, const double* Y, const double* V, double* out, int32_t r) {
  if (!c || !Y || !V || !out || r < 1 || r > XM_MAX_R) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    int64_t len = (int64_t)c->n * r;
    copy_in(c, c->hY.p, Y, len * 8);
    copy_in(c, c->hV.p, V, len * 8);
    XM_CUDA(cudaMemsetAsync(c->flags.p, 0, sizeof(int), c->stream));
    retract(c, r, c->hY.p, c->hV.p, 1.0, c->hO.p, nullptr, c->flags.p);
    int err = 0;
    XM_CUDA(cudaMemcpyAsync(&err, c->flags.p, 4, cudaMemcpyDeviceToHost, c->stream));
    copy_out(c, out, c->hO.p, len * 8);
    sync(c);
    if (err) throw Error(XM_ERETRACT, "retraction failure");
  });
}

xm_status xm_get_factor(xm_ctx* c, double* Y, int32_t* r) {
  if (!c) return XM_EINVAL;
  return guard(c, [&] {
    if (r) *r = c->r;
    if (Y && c->r > 0) copy_out(c, Y, c->Y.p, (size_t)c->n * c->r * 8);
    sync(c);
  });
}

xm_status xm_set_factor(xm_ctx* c, const double* Y, int32_t r) {
  if (!c || !Y || r < 3 || r > XM_MAX_R) return XM_EINVAL;
  return guard(c, [&] {
    require_stage(c, 1);
    c->r = r;
    copy_in(c, c->Y.p, Y, (size_t)c->n * r * 8);
    sync(c);
    c->factor_set = true;
    c->cert_valid = false;
    c->have_round = false;
  });
}

xm_status xm_get_stats(xm_ctx* c, xm_stats* out) {
  if (!c || !out) return XM_EINVAL;
  return guard(c, [&] {
    harvest_events(c);
    *out = c->stats;
  });
}

xm_status xm_set_profile(xm_ctx* c, int32_t on) {
  if (!c) return XM_EINVAL;
  return guard(c, [&] {
    harvest_events(c);
    c->opt.profile = on ? 1 : 0;  // part of the graph signature ⇒ graphs are recaptured
  });
}

xm_status xm_reset_stats(xm_ctx* c) {
  if (!c) return XM_EINVAL;
  return guard(c, [&] {
    harvest_events(c);
    int64_t E = c->stats.E, nd = c->stats.n_dup, nz = c->stats.nnzb_S, qb = c->stats.q_bytes;
    c->stats = xm_stats{};
    c->stats.E = E;
    c->stats.n_dup = nd;
    c->stats.nnzb_S = nz;
    c->stats.q_bytes = qb;
  });
}

const char* xm_last_error(xm_ctx* c) { return c ? c->last_error.c_str() : ""; }

}  // extern "C"
