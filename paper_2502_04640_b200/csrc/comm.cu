// comm.cu — NCCL over NVLink 5 / NVSwitch for the row-sharded path.
//
// The only exchange of the solve is ONE all-reduce of the n×r partial products
// after every product (one per HVP / Δf / Lanczos step): each rank streams the
// lower trapezoid of its band of Q rows (row parts of its rows, column parts of
// the rows above — spmm.cu spmm_full); all O(N·r) per-camera work and every
// dot product then run redundantly (and bitwise identically) on the replicated
// full vectors, so the inner loop needs no other collective.
// NCCL is loaded with dlopen only when world > 1 (single-GPU runs do not
// depend on it); the communicator is bootstrapped from an ncclUniqueId that
// the caller broadcasts (torch.distributed in the Python harness).
#include "xm_internal.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <map>
#include <mutex>
#include <vector>

namespace xm {

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

void load_nccl() {
  if (g_nccl.h) return;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    g_nccl.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) throw Error(XM_ENCCL, "cannot dlopen libnccl.so.2");
  auto sym = [](const char* s) {
    void* p = dlsym(g_nccl.h, s);
    if (!p) throw Error(XM_ENCCL, std::string("missing NCCL symbol ") + s);
    return p;
  };
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))sym("ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))sym("ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))sym("ncclCommDestroy");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))sym("ncclAllGather");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))sym("ncclAllReduce");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))sym("ncclGetErrorString");
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(XM_ENCCL, std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
}
}  // namespace

void nccl_unique_id(void* out128) {
  load_nccl();
  ncclUniqueId id;
  check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
}

// ---------------------------------------------------------------------------
// Loopback group: `world` contexts of ONE process (one thread each, any device)
// exchanging through device-to-device copies with host barriers.  Selected by
// an id that starts with XM_LOOPBACK_MAGIC (include/xm.h); it exists so the
// world > 1 path (sharded assembly, partial SpMM rows, padded all-gather,
// all-reduce) runs and is checked on a single-GPU box.  Same semantics as the
// NCCL calls it replaces; the all-reduce sums in rank order on every rank.
struct LoopGroup {
  int world = 0, refs = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
static std::mutex g_loop_m;
static std::map<std::string, LoopGroup*> g_loops;

static bool is_loopback_id(const void* id) {
  return id && memcmp(id, XM_LOOPBACK_MAGIC, sizeof(XM_LOOPBACK_MAGIC) - 1) == 0;
}

void nccl_init(xm_ctx* c, const void* id) {
  if (c->world <= 1) return;
  if (!id) throw Error(XM_EINVAL, "world > 1 requires an ncclUniqueId");
  if (is_loopback_id(id)) {
    std::string key((const char*)id, 128);
    std::lock_guard<std::mutex> lk(g_loop_m);
    LoopGroup*& g = g_loops[key];
    if (!g) {
      g = new LoopGroup();
      g->world = c->world;
      g->ptr.assign(c->world, nullptr);
    }
    if (g->world != c->world) throw Error(XM_EINVAL, "loopback group: world mismatch");
    ++g->refs;
    c->loop = g;
    c->loop_key = key;
    return;
  }
  load_nccl();
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  check(g_nccl.CommInitRank(&comm, c->world, uid, c->rank), "ncclCommInitRank");
  c->nccl_comm = comm;
}

void nccl_destroy(xm_ctx* c) {
  if (c->loop) {
    std::lock_guard<std::mutex> lk(g_loop_m);
    LoopGroup* g = static_cast<LoopGroup*>(c->loop);
    if (--g->refs == 0) {
      g_loops.erase(c->loop_key);
      delete g;
    }
    c->loop = nullptr;
  }
  if (c->nccl_comm && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)c->nccl_comm);
  c->nccl_comm = nullptr;
}

void nccl_allreduce_sum(xm_ctx* c, double* buf, size_t count) {
  if (c->world <= 1) return;
  if (c->loop) {
    LoopGroup* g = static_cast<LoopGroup*>(c->loop);
    std::vector<double> all((size_t)c->world * count), sum(count, 0.0);
    XM_CUDA(cudaStreamSynchronize(c->stream));
    g->ptr[c->rank] = buf;
    g->barrier();
    for (int q = 0; q < c->world; ++q)
      XM_CUDA(cudaMemcpy(all.data() + (size_t)q * count, g->ptr[q], count * 8, cudaMemcpyDefault));
    g->barrier();
    for (int q = 0; q < c->world; ++q)
      for (size_t k = 0; k < count; ++k) sum[k] += all[(size_t)q * count + k];
    XM_CUDA(cudaMemcpy(buf, sum.data(), count * 8, cudaMemcpyDefault));
    return;
  }
  check(g_nccl.AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm,
                         c->stream),
        "ncclAllReduce");
}

// recv[q·count … (q+1)·count) = rank q's send (count doubles per rank)
void nccl_allgather_f64(xm_ctx* c, const double* send, double* recv, size_t count) {
  if (c->world <= 1) {
    if (recv != send) XM_CUDA(cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, c->stream));
    return;
  }
  if (c->loop) {
    LoopGroup* g = static_cast<LoopGroup*>(c->loop);
    XM_CUDA(cudaStreamSynchronize(c->stream));
    g->ptr[c->rank] = send;
    g->barrier();
    for (int q = 0; q < c->world; ++q)
      XM_CUDA(cudaMemcpy(recv + (size_t)q * count, g->ptr[q], count * 8, cudaMemcpyDefault));
    g->barrier();
    return;
  }
  check(g_nccl.AllGather(send, recv, count, ncclFloat64, (ncclComm_t)c->nccl_comm, c->stream),
        "ncclAllGather");
}

}  // namespace xm
