// blas.cu — cuBLAS for the plain dense fp64 GEMM / SYRK updates of the Q
// assembly (H5: G = L⁻¹C̄ block updates, Q = S − GᵀG) and of the blocked
// Cholesky factorisations (K̄, and Z + εI in the PSD test).  These are plain
// library GEMMs, not the streaming hot path ("cuBLAS only for
// plain library GEMMs"); the diagonal-block factorisations and triangular
// solves stay hand-written (assembly.cu).  cuBLAS is dlopen'ed (like NCCL), one
// handle per context on the context's stream; if it cannot be loaded the
// library's own k_dgemm runs instead (GPU either way).
//
// Row-major ↔ column-major: a row-major M×N matrix with leading dimension ld
// is the column-major N×M matrix Xᵀ with the same ld, so
//   C = α·op(A)·op(B) + βC   (row-major)   ⇔   Cᵀ = α·op(B)ᵀ·op(A)ᵀ + βCᵀ.
#include "xm_internal.cuh"

#include <cublas_v2.h>
#include <dlfcn.h>

#include <mutex>

namespace xm {

namespace {
struct CublasApi {
  void* h = nullptr;
  bool tried = false;
  cublasStatus_t (*Create)(cublasHandle_t*) = nullptr;
  cublasStatus_t (*Destroy)(cublasHandle_t) = nullptr;
  cublasStatus_t (*SetStream)(cublasHandle_t, cudaStream_t) = nullptr;
  cublasStatus_t (*Dgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                          const double*, const double*, int, const double*, int, const double*,
                          double*, int) = nullptr;
  cublasStatus_t (*Dsyrk)(cublasHandle_t, cublasFillMode_t, cublasOperation_t, int, int,
                          const double*, const double*, int, const double*, double*, int) = nullptr;
};
CublasApi g_blas;
std::mutex g_blas_m;

bool load_cublas() {
  std::lock_guard<std::mutex> lk(g_blas_m);
  if (g_blas.tried) return g_blas.h != nullptr;
  g_blas.tried = true;
  if (std::getenv("XM_NO_CUBLAS")) return false;
  for (const char* nm : {"libcublas.so.12", "libcublas.so"}) {
    g_blas.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_blas.h) break;
  }
  if (!g_blas.h) return false;
  g_blas.Create = (decltype(g_blas.Create))dlsym(g_blas.h, "cublasCreate_v2");
  g_blas.Destroy = (decltype(g_blas.Destroy))dlsym(g_blas.h, "cublasDestroy_v2");
  g_blas.SetStream = (decltype(g_blas.SetStream))dlsym(g_blas.h, "cublasSetStream_v2");
  g_blas.Dgemm = (decltype(g_blas.Dgemm))dlsym(g_blas.h, "cublasDgemm_v2");
  g_blas.Dsyrk = (decltype(g_blas.Dsyrk))dlsym(g_blas.h, "cublasDsyrk_v2");
  if (!g_blas.Create || !g_blas.Destroy || !g_blas.SetStream || !g_blas.Dgemm || !g_blas.Dsyrk) {
    g_blas.h = nullptr;
    return false;
  }
  return true;
}

cublasHandle_t handle(xm_ctx* c) {
  if (!c->cublas) {
    cublasHandle_t h = nullptr;
    if (g_blas.Create(&h) != CUBLAS_STATUS_SUCCESS) throw Error(XM_ECUDA, "cublasCreate failed");
    c->cublas = h;
  }
  cublasHandle_t h = static_cast<cublasHandle_t>(c->cublas);
  if (g_blas.SetStream(h, c->stream) != CUBLAS_STATUS_SUCCESS)
    throw Error(XM_ECUDA, "cublasSetStream failed");
  return h;
}

void check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) throw Error(XM_ECUDA, std::string(what) + " failed");
}
}  // namespace

bool blas_dgemm(xm_ctx* c, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  if (!load_cublas()) return false;
  check(g_blas.Dgemm(handle(c), tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, N, M,
                     K, &alpha, B, (int)ldb, A, (int)lda, &beta, C, (int)ldc),
        "cublasDgemm");
  return true;
}

// Row-major lower triangle of C (n×n) ← β·C + α·X·Xᵀ, X row-major n×k (trans_x
// = false) or α·Xᵀ·X, X row-major k×n (trans_x = true).
bool blas_dsyrk_lower(xm_ctx* c, bool trans_x, int n, int k, double alpha, const double* X,
                      int64_t ldx, double beta, double* C, int64_t ldc) {
  if (!load_cublas()) return false;
  // column-major view: X_cm = X_rmᵀ; row-major lower of C = column-major upper
  //   X·Xᵀ  = X_cmᵀ·X_cm  → trans = T;   Xᵀ·X = X_cm·X_cmᵀ → trans = N
  check(g_blas.Dsyrk(handle(c), CUBLAS_FILL_MODE_UPPER, trans_x ? CUBLAS_OP_N : CUBLAS_OP_T, n, k,
                     &alpha, X, (int)ldx, &beta, C, (int)ldc),
        "cublasDsyrk");
  return true;
}

void blas_destroy(xm_ctx* c) {
  if (c->cublas && g_blas.Destroy) g_blas.Destroy(static_cast<cublasHandle_t>(c->cublas));
  c->cublas = nullptr;
}

}  // namespace xm
