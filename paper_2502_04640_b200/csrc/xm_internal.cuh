// xm_internal.cuh — shared declarations of libxm (B200 / sm_100a, fp64).
//
// Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; SURVEY §8 rows H1..H13.
// Nothing here is shared with oracle/ (the CPU oracle is independent).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/xm.h"
#include <nvtx3/nvToolsExt.h>

#define XM_MAX_R 12

namespace xm {

// ---------------------------------------------------------------- errors
struct Error : public std::runtime_error {
  xm_status code;
  Error(xm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define XM_CUDA(call)                                                                \
  do {                                                                               \
    cudaError_t e__ = (call);                                                        \
    if (e__ != cudaSuccess)                                                          \
      throw ::xm::Error(XM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

#define XM_CHECK_LAUNCH() XM_CUDA(cudaGetLastError())

// NVTX range for profilers (nsys / ncu --nvtx); no-op without an attached tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- device buffers
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw Error(XM_ENOMEM, "cudaMalloc " + std::to_string(count * sizeof(T)) + " bytes");
    }
    n = count;
  }
  operator T*() const { return p; }
  T* get() const { return p; }
};

// ---------------------------------------------------------------- tCG device state
// All trust-region / tCG scalars live in device memory so that the inner loop
// can run without host round trips (kernels read α, β, τ from here).
struct TcgState {
  double Delta;      // TR radius
  double z, z_old, r0, e_Pe, e_Pd, d_Pd;
  double alpha, beta, tau, d_Hd, e_Pe_new;
  double kappa, theta;
  int j;             // completed iterations
  int max_inner;
  int stop;          // 0 running, 1 negcurv, 2 exceeded, 3 converged, 4 maxinner
  int boundary;      // this iteration steps to the TR boundary
  int n_hvp;
  int pad;
};

enum { TCG_RUNNING = 0, TCG_NEGCURV = 1, TCG_EXCEEDED = 2, TCG_CONVERGED = 3, TCG_MAXINNER = 4 };

// ---------------------------------------------------------------- launch helpers
struct Launcher;  // fwd

}  // namespace xm

// The context (opaque in the ABI).
namespace xm {
constexpr int kPinD = 0, kPinTcg = 16, kPinDoubles = 512;
}
struct xm_ctx {
  int device = 0, rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  xm_options opt{};
  xm_stats stats{};
  int stage = 0;  // 0 created, 1 Q built, 2 solved

  // problem
  int N = 0, M = 0;
  int64_t E = 0;      // after de-duplication
  int64_t E_user = 0; // measurements in the caller's last xm_build_Q input (XM² maps back to it)
  int n = 0;          // 3N
  int64_t ldq = 0;    // leading dimension of Q / G rows (padded to 32 doubles)
  int64_t ldk = 0;    // leading dimension of K̄ / L
  // sharding: frames [f0, f1) → rows [row0, row0 + nrows)
  int nfpr = 0, f0 = 0, f1 = 0, row0 = 0, nrows = 0;
  double normQ = 0.0, normQ2_local = 0.0;

  // canonical edges (sorted by (landmark, frame))
  xm::DBuf<int32_t> e_fr, e_lm;
  xm::DBuf<int32_t> e_in;     // canonical measurement → index in the last build's input
  xm::DBuf<int32_t> orig_in;  // XM² rebuilds: build-input index → caller's index (empty: identity)
  xm::DBuf<double> e_pts, e_w;
  xm::DBuf<int32_t> lm_off, fr_off, fr_edge;  // track / frame offsets, frame-sorted edge ids
  xm::DBuf<double> W;                        // per-landmark weight Σ w_e (Q_3 diag)
  // S pattern
  xm::DBuf<int64_t> s_rowptr;
  xm::DBuf<int32_t> s_colidx;
  int64_t nnzb = 0;
  bool pattern_valid = false;  // S pattern built (eagerly with dense Q, on demand matrix-free)
  // dense assembly products
  xm::DBuf<double> Q;   // nrows × ldq (this rank's rows)
  xm::DBuf<double> L;   // (N−1) × ldk  Cholesky of K̄
  xm::DBuf<double> G;   // (N−1) × ldq  L⁻¹ C̄
  bool have_recovery = false;  // L, G valid (false after xm_set_Q)

  // solver state (all n_alloc × r row-major, replicated on every rank)
  int r = 0;
  int64_t n_alloc = 0;  // rows allocated for vectors (≥ world·3·nfpr)
  xm::DBuf<double> Y, QY, grad, eta, Heta, res, dir, Hdir, Ynew, Dv, QD, tmp, tmp2;
  xm::DBuf<double> alpha;  // N
  xm::DBuf<double> regd;   // N: App. D diagonal shifts d_i = 2λ/3 (α_i − 1) at the current factor
  // NEXT-1 matrix-free mode (implicit.cu): frame-sorted measurement copies, K̄⁻¹
  bool implicit_active = false;
  xm::DBuf<int32_t> imp_lm;                // frame-sorted landmark ids
  xm::DBuf<double> imp_pts, imp_w, Kinv;   // w·ũ (landmark- and frame-sorted SoA), frame-sorted w
  xm::DBuf<double> imp_mom, imp_tb;        // per-frame c_i, A_i; [0; K̄⁻¹ b]
  void* imp_sym_plan = nullptr;            // lower-triangle stream plan of K̄⁻¹
  // world > 1: this rank's landmarks [k0, k1), frames [f0, f1), K̄⁻¹ rows [ka, kb)
  int imp_k0 = 0, imp_k1 = 0, imp_f0 = 0, imp_f1 = 0, imp_ka = 0, imp_kb = 0;
  int64_t imp_el = 0, imp_ef = 0;  // measurements of this rank's landmarks / frames
  xm::DBuf<double> imp_sym_part;
  xm::DBuf<double> lam;    // N × 6 (xx, yy, zz, xy, xz, yz)
  xm::DBuf<double> part;   // SpMM split-K partials: nsplit × nrows × r
  xm::DBuf<double> red;    // block partials for reductions
  xm::DBuf<double> scal;   // reduced scalars (device)
  xm::DBuf<xm::TcgState> tcg;   // [2]: double-buffered tCG state
  xm::DBuf<double> part1, part2; // scalar partials of the tCG kernels
  xm::DBuf<int> flags;     // error flags etc.
  xm::DBuf<double> hostbuf_dummy;
  double* h_scal = nullptr;  // pinned host mirror of scal
  xm::TcgState* h_tcg = nullptr;
  int* h_flags = nullptr;
  bool factor_set = false;
  // Lanczos
  xm::DBuf<double> lz_V, lz_w, lz_c, lz_part, lz_x;
  double last_lambda = 0.0;
  int last_lanczos_steps = 0;
  bool have_cert = false;
  xm_certificate cert{};
  xm_solve_info info{};
  // rounding
  xm::DBuf<double> Yr;  // n × 3 rounded factor
  xm::DBuf<double> Rs;  // N × 9, s N, t N×3, p M×3
  xm::DBuf<double> s_out, t_out, p_out, rhs;
  int n_flipped = 0;
  bool have_round = false;
  // profiling
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  xm::DBuf<int> ev_exec;           // per event pair: 1 if the SpMM actually ran
  std::vector<double> ev_bytes;    // per event pair: algorithmic bytes
  // NCCL (or the in-process loopback group used to test world > 1 on one GPU)
  void* nccl_comm = nullptr;
  void* loop = nullptr;
  std::string loop_key;
  // lower-triangle SpMM work plan + tensor map (spmm_sym.cu)
  void* sym_plan = nullptr;
  xm::DBuf<double> gbuf;  // all-gather staging
  // hooks (test / bench entry points) use their own scratch
  xm::DBuf<double> hY, hV, hO, hQY;
  // certificate cache (valid while the factor is unchanged)
  bool cert_valid = false;
  double cert_lambda = 0.0;
  int cert_steps = 0;
  xm::DBuf<double> cert_v;
  xm::DBuf<double> Zw;       // Z + εI work copy for the Cholesky PSD test
  double cert_lower = 0.0;   // certified lower bound on λ_min(Z)
  int cert_method = 0;       // 0 Lanczos converged, 1 Cholesky of Z + εI + shift-invert Lanczos
  int cert_rigorous = 0;     // 1: cert_lower proven by a completed Cholesky
  int tcg_batch = 8;
  // CUDA graph of `tcg_batch` tCG iterations per rank r (captured once, replayed)
  struct TcgGraph {
    cudaGraphExec_t exec = nullptr;
    int batch = 0;                                // iterations per replay (0: conditional loop)
    bool loop = false;                            // conditional WHILE node: the whole tCG per replay
    int64_t launches = 0, spmms = 0;              // kernels / SpMMs per replay (loop: per iteration)
    std::vector<cudaEvent_t> ev;                  // profiling event pairs (captured)
    std::vector<double> bytes;                    // algorithmic bytes per pair
    xm::DBuf<int> execf;                          // per pair: 1 if the SpMM ran
    std::vector<uintptr_t> sig;                   // buffers / sizes the capture baked in
  };
  TcgGraph tcg_graphs[XM_MAX_R + 1];
  // the outer iteration's step after tCG (retraction, Δf product, dots) as one
  // graph per rank r (profile off, one GPU)
  TcgGraph post_graphs[XM_MAX_R + 1];
  TcgGraph* cap_target = nullptr;                 // non-null while capturing
  // capturing the body of a conditional WHILE node (the whole tCG loop in one
  // graph launch): k_tcg_dir clears `cap_cond` when the tCG state says stop
  cudaGraphConditionalHandle cap_cond = 0;
  bool cap_cond_on = false;
  cudaStream_t cap_stream = nullptr;
  // side stream + events of the look-ahead Cholesky (assembly.cu dense_cholesky)
  cudaStream_t aux_stream = nullptr;
  // pinned host scalars: several device → host reads completed by ONE sync
  // (kPinD: the outer iteration's Δf terms; kPinTcg: a deferred tCG state)
  double* hpin = nullptr;
  int64_t tcg_defer_launches = 0;
  cudaEvent_t ev_la = nullptr, ev_lb = nullptr;
  // TRSM: the super-block inverses L_ss⁻¹ (independent of the right-hand side)
  // are computed ahead on kTrsmStreams forked streams (dense_trsm_lower_left)
  static constexpr int kTrsmStreams = 4;
  cudaStream_t trsm_streams[kTrsmStreams] = {};
  cudaEvent_t trsm_ev[kTrsmStreams + 1] = {};
  bool use_graphs = true;
  xm::DBuf<double> sym_part;       // per-unit row / column partials of the symmetric SpMM
  // XM_PHASES=1: host wall-clock breakdown of xm_solve (synchronises; diagnostics only)
  bool phases_on = false;
  bool fused_tcg = true;    // XM_NO_FUSED_TCG=1: three-kernel tCG iteration (A/B measurement)
  bool persist_tcg = true;
  int gemm_tile = 0;        // XM_GEMM_TILE=bk16|mid: A/B variants of the DMMA tile for K > 64
  int trsm_sb = 512;        // XM_TRSM_SB: TRSM super-block rows (multiple of 64)  // XM_NO_PERSIST_TCG=1: one launch per tCG iteration instead
  int persist_sym = 0;      // lower-triangle persistent tCG: 0 auto (N < 4000), 1 forced (XM_SYM_TCG), -1 off (XM_NO_SYM_TCG)
  void* persist_sym_plan = nullptr;
  xm::DBuf<double> dir2;    // δ ping-pong partner of dir (persistent tCG)
  cudaEvent_t ev_persist[2] = {nullptr, nullptr};
  // persistent tCG: 2-D tensor map of Q (box 128 columns × bh rows), raw CUtensorMap bytes
  alignas(64) unsigned char persist_tmap[128] = {0};
  const void* persist_tmap_q = nullptr;
  int persist_tmap_bh = 0, persist_tmap_n = 0;
  xm::DBuf<unsigned long long> tdbg;  // XM_PHASES: fused-tCG phase stamps
  double phase_ms[8] = {0};
  long long phase_n[8] = {0};
  xm::DBuf<int> gbar;                  // software grid-barrier state of the symmetric SpMM
  xm::DBuf<unsigned long long> gsync;  // fused tCG grid_sync counter (reset by tcg_init)
  // named scratch buffers that persist across calls (grow-only): no cudaMalloc /
  // cudaFree churn (each cudaFree synchronises the device) inside build / solve
  std::map<std::string, xm::DBuf<int32_t>> s_i32;
  std::map<std::string, xm::DBuf<uint32_t>> s_u32;
  std::map<std::string, xm::DBuf<uint64_t>> s_u64;
  std::map<std::string, xm::DBuf<int64_t>> s_i64;
  std::map<std::string, xm::DBuf<double>> s_f64;
  std::string last_error;
};

namespace xm {

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
inline int64_t round_up(int64_t a, int64_t b) { return ((a + b - 1) / b) * b; }

// Pointer helpers: copy between caller memory (host or device) and device.
bool is_device_ptr(const void* p);
void copy_in(xm_ctx* c, void* dst_dev, const void* src, size_t bytes);
void copy_out(xm_ctx* c, void* dst, const void* src_dev, size_t bytes);
void sync(xm_ctx* c);
inline void count_launch(xm_ctx* c, int k = 1) { c->stats.kernel_launches += k; }

// cudaFuncAttributeMaxDynamicSharedMemorySize for `kern` on the CURRENT device
// (the attribute is per device context).  Cached per (thread, device, kernel):
// no process-wide flag, so independent contexts on other devices / threads
// (loopback ranks) each set it for themselves.
void ensure_smem_attr(const void* kern, size_t smem);

// Persistent named scratch (see xm_ctx::s_*).
inline DBuf<int32_t>& scratch_i32(xm_ctx* c, const std::string& k) { return c->s_i32[k]; }
inline DBuf<uint32_t>& scratch_u32(xm_ctx* c, const std::string& k) { return c->s_u32[k]; }
inline DBuf<uint64_t>& scratch_u64(xm_ctx* c, const std::string& k) { return c->s_u64[k]; }
inline DBuf<int64_t>& scratch_i64(xm_ctx* c, const std::string& k) { return c->s_i64[k]; }
inline DBuf<double>& scratch_f64(xm_ctx* c, const std::string& k) { return c->s_f64[k]; }

// ------------------------------------------------------------ util kernels (util.cu)
// Deterministic reductions: blocks write partials, one block reduces in fixed order.
// min_mask: bit c set ⇒ component c is reduced with min instead of sum.
void reduce_partials(xm_ctx* c, const double* partials, int nblk, int ncomp, double* out,
                     unsigned min_mask = 0u);
void exclusive_scan_i32(xm_ctx* c, const int32_t* in, int32_t* out, int64_t n, int32_t* total_dev);
void radix_sort_u64(xm_ctx* c, uint64_t* keys, uint32_t* vals, int64_t n, int bits,
                    DBuf<uint64_t>& tmp_k, DBuf<uint32_t>& tmp_v);
void dot2_flat(xm_ctx* c, const double* a0, const double* b0, const double* a1, const double* b1,
               int64_t len, double* partials, int nblk);
void dot_flat(xm_ctx* c, const double* a, const double* b, int64_t len, double* partials, int nblk);
constexpr int kDotBlocks = 296;  // 2 × 148 SMs; fixed ⇒ deterministic sums

// ------------------------------------------------------------ assembly (assembly.cu)
void build_Q_device(xm_ctx* c, int N, int M, int64_t E, const int32_t* fr, const int32_t* lm,
                    const double* pts, const double* w);
bool dense_cholesky(xm_ctx* c, double* A, int m, int64_t lda, double rel_tol,
                    bool throw_on_fail = true, double* U = nullptr, int64_t ldu = 0);
bool psd_test_cholesky(xm_ctx* c, double shift, double* lower = nullptr, double* U = nullptr,
                       int64_t ldu = 0);
void dense_trsm_lower_left(xm_ctx* c, const double* L, int m, int64_t ldl, const double* U,
                           int64_t ldu, double* B, int ncols, int64_t ldb, bool lower_rhs = false);
// C (lower tiles) = α XᵀX + β C for lower-triangular X (k-loop from the tile row)
void dsyrk_tn_lowtri(xm_ctx* c, int M, double alpha, const double* X, int64_t ldx, double beta, double* C,
                     int64_t ldc);
// C = β·C + α·Σ_k A[k·lda + m]·B[k·ldb + n] on the fp64 tensor cores (dgemm_tn.cu);
// lower ⇒ only the lower-triangle tiles (M == N)
void dgemm_tn(xm_ctx* c, bool lower, int M, int N, int K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc);
void mirror_lower(xm_ctx* c, double* Q, int n, int64_t ldq);
void identity(xm_ctx* c, double* A, int n, int64_t lda);  // A ← I (n×n, row-major)

// ------------------------------------------------------------ SpMM (spmm.cu)
enum { EPI_STORE = 0, EPI_HVP = 1, EPI_ZMUL = 2, EPI_DF = 3, EPI_GRAD = 4, EPI_TCG = 5 };
struct GridBar {  // sense-reversing software grid barrier state (frame_ops.cuh)
  int count;
  int sense;
};
struct SpmmEpiArgs {
  double* out = nullptr;         // STORE / ZMUL (Zv) / DF (QD) / GRAD (QY): full-layout rows
  double* out2 = nullptr;        // HVP: Hv;  GRAD: grad
  const double* Y = nullptr;     // HVP: current point
  const double* lam = nullptr;   // HVP / ZMUL: Λ (N × 6)
  const double* aux = nullptr;   // DF: QY
  double* lam_out = nullptr;     // GRAD: Λ written here
  double* partials = nullptr;    // per-CTA scalar partials [G][NC]
  const int* stop = nullptr;     // no-op when *stop != 0
  int* exec = nullptr;           // profiling: set to 1 when the kernel ran
  // EPI_TCG (one fused Steihaug–Toint iteration, world == 1): V = δ (updated
  // in place), partials = ⟨δ,Hδ⟩ per CTA, p2 = ‖r‖² per CTA, st = state
  TcgState* st = nullptr;
  double* eta = nullptr;
  double* Heta = nullptr;
  double* res = nullptr;
  double* p2 = nullptr;
  GridBar* gbar = nullptr;
  unsigned long long* dbg = nullptr;  // XM_PHASES: per-CTA %globaltimer stamps [G][8]
  unsigned long long* gsync = nullptr;  // EPI_TCG: grid_sync arrival counter
};
int spmm_grid(xm_ctx* c, int r);  // number of scalar partials written by spmm()
bool spmm_sym_supported(xm_ctx* c, int r);
bool tcg_fused_supported(xm_ctx* c, int r);  // one-launch tCG iteration (EPI_TCG)
bool tcg_persist_supported(xm_ctx* c, int r);  // whole tCG solve in one launch
bool tcg_persist_sym_supported(xm_ctx* c, int r);  // ... with the lower-triangle stream
void tcg_persist_launch(xm_ctx* c, int r);
double tcg_persist_bytes_per_iter(xm_ctx* c, int r);
int spmm_sym_partials(xm_ctx* c);
bool tcg_fullrow_ok(xm_ctx* c);  // tCG may use the full-row fused / persistent kernels
void spmm_sym_launch(xm_ctx* c, const double* V, int r, int mode, const SpmmEpiArgs& ep);
void spmm(xm_ctx* c, const double* V, int r, int mode, const SpmmEpiArgs& ep);
// Full product into out (n × r, replicated): this rank's rows + all-gather.
void spmm_full(xm_ctx* c, const double* V, int r, double* out_full, const int* stop = nullptr);
void harvest_events(xm_ctx* c);

// ------------------------------------------------------------ manifold (manifold.cu)
// grad = 2(QY − ΛY); Λ written to c->lam; scal_out[0..2] = f, ‖g‖², min α (i ≥ 1).
void grad_and_multipliers(xm_ctx* c, int r, const double* Y, const double* QY, double* grad,
                          double* scal_out /*3*/);
void project(xm_ctx* c, int r, const double* Y, const double* W, double* out);
// Y_out = R_Y(step·V); D = Y_out − Y (nullable); optional partials of ⟨g, V⟩ and
// ⟨V, HV⟩ (dots2 != nullptr) written as [nblk][2].
void retract(xm_ctx* c, int r, const double* Y, const double* V, double step, double* Yout,
             double* D, int* err, const double* g = nullptr, const double* HV = nullptr,
             double* dots2 = nullptr);
// HV = P(2·QV − 2ΛV), partials of ⟨V, HV⟩ (one per block of 128 cameras).
void hvp_epilogue(xm_ctx* c, int r, const double* Y, const double* V, const double* QV,
                  double* HV, double* partials, const int* stop);
int frame_blocks(xm_ctx* c);
// Hessian-vector product V → HV with ⟨V,HV⟩ partials; returns the partial count.
int hvp_product(xm_ctx* c, int r, const double* Y, const double* V, double* HV, double* partials,
                const int* stop);
// tCG with double-buffered device state st[0] / st[1] (TcgState)
void tcg_init(xm_ctx* c, int r, double Delta);
void tcg_iteration(xm_ctx* c, int r);
void axpy(xm_ctx* c, int64_t len, double a, const double* x, double* y);
void pad_column(xm_ctx* c, int r, const double* Y, double* Yz, const double* v, double* Dz);
void zmul(xm_ctx* c, const double* x, const double* Zx_q, double* out);  // Zx = Qx − Λx (r = 1)
// NEXT-4 (batch.cu)
size_t batch_smem_bytes(int N, int lanczos_max);
void batch_staircase(xm_ctx* c, int B, int N, const double* Q_dev, int64_t qstride,
                     const double* Y0_dev, int r0, double* Yout_dev, xm_batch_result* res_dev);
// NEXT-1 (implicit.cu)
void implicit_prepare(xm_ctx* c);
void build_s_pattern(xm_ctx* c, int N);
bool prefer_implicit(int N, int64_t E, int world);
void implicit_product(xm_ctx* c, const double* V, int r, double* out, const int* stop = nullptr,
                      int* exec = nullptr);
double implicit_alg_bytes(xm_ctx* c, int r);
void implicit_translations(xm_ctx* c, const double* Y3, double* t_out);
double implicit_normF(xm_ctx* c);
void splitmix_uniform(xm_ctx* c, int64_t n, uint64_t seed, double* out);  // cert.cu
// products may use the dense fused kernels (one GPU, Q formed) / fused epilogues too (no App. D)
inline bool dense_fused(xm_ctx* c) { return c->world == 1 && !c->implicit_active; }
inline bool fused_epilogues(xm_ctx* c) { return dense_fused(c) && c->opt.scale_reg == 0.0; }
// App. D (scale_reg λ): scal_out[0] = F(Y), [1] = Σ_{i≥1}(α_i² − 1), [2] = F(Y+D) − F(Y) (D may
// be NULL); d_i = 2λ/3 (α_i − 1) into c->regd
void reg_frames(xm_ctx* c, int r, const double* Y, const double* D, double* scal_out);

// ------------------------------------------------------------ Lanczos / rounding (cert.cu)
// returns true if the smallest Ritz pair converged (|β_k s_k| ≤ tol_abs)
struct LanczosOp {
  const double* X = nullptr;  // non-null: shift-invert operator −XᵀX (X = L⁻¹ lower, row-major)
  int64_t ldx = 0;
};
bool lanczos(xm_ctx* c, double tol_abs, int max_steps, double* lambda, int* steps,
             double* vec_dev, const LanczosOp& op = LanczosOp());
void round_recover_device(xm_ctx* c);
// xm2.cu
void edge_residuals_user(xm_ctx* c, double* out_dev);
void xm2_device(xm_ctx* c, double frac, uint8_t* keep_user_dev, int64_t* n_dropped, int64_t* n_restored);

// ------------------------------------------------------------ NCCL (comm.cu)
void nccl_unique_id(void* out128);
void nccl_init(xm_ctx* c, const void* id);
void nccl_destroy(xm_ctx* c);
void nccl_allreduce_sum(xm_ctx* c, double* buf, size_t count);
void nccl_allgather_f64(xm_ctx* c, const double* send, double* recv, size_t count);
void sym_plan_destroy(xm_ctx* c);
void sym_plan_slot_destroy(void*& slot);
void spmm_sym_matrix(xm_ctx* c, void*& plan_slot, DBuf<double>& part, const double* A, int m,
                     int64_t lda, const double* V, int r, double* out, const int* stop, int row0 = 0,
                     int nrows = -1);
void sym_tcg_plan_destroy(xm_ctx* c);

// Row sharding: rank q owns frames [q·nfpr, min(N, (q+1)·nfpr)),
// nfpr = ⌈N/world⌉; vectors exchanged by the all-gather hold world·3·nfpr rows.
// Row bands of the world > 1 layout (composed with the
// lower-triangle stream): rank p owns frames [F_p, F_{p+1}) and stores only
// the lower trapezoid of their rows (columns ≤ row).  Its share of the lower
// triangle is ∝ F_{p+1}² − F_p², so F_p = N·√(p/world) balances the bytes per
// product; bands are aligned to 32 frames (= 96 rows = 3 tiles of 32 rows, so
// the streaming kernel's tiles never straddle two ranks).  nfpr = the largest
// band (buffer sizing).
inline int band_start(int N, int world, int p) {
  if (p <= 0) return 0;
  if (p >= world) return N;
  const double x = (double)N * std::sqrt((double)p / (double)world);
  const int a = (int)std::lround(x / 32.0) * 32;
  return std::min(N, std::max(0, a));
}
inline void shard_of(int N, int world, int rank, int* f0, int* f1, int* nfpr) {
  *f0 = band_start(N, world, rank);
  *f1 = std::max(*f0, band_start(N, world, rank + 1));
  int m = 0;
  for (int p = 0; p < world; ++p)
    m = std::max(m, band_start(N, world, p + 1) - band_start(N, world, p));
  *nfpr = std::max(m, 1);
}
inline void set_shard(xm_ctx* c, int N) {
  shard_of(N, c->world, c->rank, &c->f0, &c->f1, &c->nfpr);
  c->row0 = 3 * c->f0;
  c->nrows = 3 * (c->f1 - c->f0);
}

}  // namespace xm
