// Library-owned NCCL communicator (north_star: destination-partitioned graph,
// projected source features exchanged with NCCL all-gather over NVLink).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: in a PyTorch process this resolves to the
// NCCL torch already loaded), so librgnn itself loads on machines without NCCL and only the comm
// entry points report RGNN_ERR_NCCL there.  The paper has no multi-GPU path (§3.6.2,
// "We focused Hector on single-GPU performance"); this follows SURVEY.md §8(e) variant X.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "comm.cuh"

namespace rgnn {
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer an NCCL already in the process (PyTorch's), then the loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    a.h = h;
    bool ok = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        ok = false;
        a.err += std::string(a.err.empty() ? "" : ", ") + "missing " + name;
      }
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.Reduce, "ncclReduce");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    if (!ok) a.h = nullptr;
  });
  RGNN_CHECK(a.h != nullptr, RGNN_ERR_NCCL, a.err);
  return a;
}

#define RGNN_NCCL(call)                                                                                   \
  do {                                                                                                    \
    ncclResult_t r_ = (call);                                                                             \
    if (r_ != ncclSuccess)                                                                                \
      RGNN_FAIL(RGNN_ERR_NCCL, std::string(#call) + ": " + api().GetErrorString(r_));                     \
  } while (0)

}  // namespace

// ---------------------------------------------------------------- exchange steps
// Forward all-gather of the node rows (variant X of SURVEY.md §8(e)), in place and chunked by owner:
// one ncclBroadcast per root rank k of its rows [node_ptr[k], node_ptr[k+1]) (uneven ranges), each
// followed by an event, all on the comm stream after `s` has produced this rank's rows.  The compute
// stream waits on chunk k's event only before the work that gathers rows of chunk k (the pair GEMM
// tiles of those sources), so the transfer of chunk k+1 overlaps the GEMM of chunk k.
void comm_allgather_rows_begin(rgnn_comm_s* c, void* rows, size_t row_bytes, cudaStream_t s) {
  NcclApi& a = api();
  RGNN_CUDA(cudaEventRecord(c->start, s));
  RGNN_CUDA(cudaStreamWaitEvent(c->cs, c->start, 0));
  char* base = static_cast<char*>(rows);
  for (int k = 0; k < c->world; ++k) {
    const size_t off = (size_t)c->node_ptr[k] * row_bytes;
    const size_t n = (size_t)(c->node_ptr[k + 1] - c->node_ptr[k]) * row_bytes;
    if (n) RGNN_NCCL(a.Broadcast(base + off, base + off, n, ncclInt8, k, c->nc, c->cs));
    RGNN_CUDA(cudaEventRecord(c->chunk[k], c->cs));
  }
}

void comm_wait_chunk(rgnn_comm_s* c, int k, cudaStream_t s) {
  if (k != c->rank) RGNN_CUDA(cudaStreamWaitEvent(s, c->chunk[k], 0));
}

void comm_wait_all(rgnn_comm_s* c, cudaStream_t s) {
  for (int k = 0; k < c->world; ++k) comm_wait_chunk(c, k, s);
}

// Backward exchange: the partial dX of every source row (this rank's pair contributions) summed
// onto the owner of each row range (a reduce-scatter with uneven counts: one in-place ncclReduce per
// root), and every weight gradient summed on all ranks (ncclAllReduce, in place); one NCCL group on
// the comm stream, joined back into `s`.
void comm_reduce_grads(rgnn_comm_s* c, float* dX, int64_t d_in, const std::vector<std::pair<float*, size_t>>& dW,
                       cudaStream_t s) {
  NcclApi& a = api();
  RGNN_CUDA(cudaEventRecord(c->start, s));
  RGNN_CUDA(cudaStreamWaitEvent(c->cs, c->start, 0));
  RGNN_NCCL(a.GroupStart());
  if (dX)
    for (int k = 0; k < c->world; ++k) {
      const size_t off = (size_t)c->node_ptr[k] * d_in;
      const size_t n = (size_t)(c->node_ptr[k + 1] - c->node_ptr[k]) * d_in;
      if (n) RGNN_NCCL(a.Reduce(dX + off, dX + off, n, ncclFloat32, ncclSum, k, c->nc, c->cs));
    }
  for (const auto& w : dW)
    if (w.first && w.second) RGNN_NCCL(a.AllReduce(w.first, w.first, w.second, ncclFloat32, ncclSum, c->nc, c->cs));
  RGNN_NCCL(a.GroupEnd());
  RGNN_CUDA(cudaEventRecord(c->done, c->cs));
  RGNN_CUDA(cudaStreamWaitEvent(s, c->done, 0));
}

void comm_join(rgnn_comm_s* c, cudaStream_t s) {
  RGNN_CUDA(cudaEventRecord(c->done, c->cs));
  RGNN_CUDA(cudaStreamWaitEvent(s, c->done, 0));
}

}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_comm_unique_id(void* id_out) {
  return guarded([&] {
    RGNN_CHECK(id_out, RGNN_ERR_INVALID_ARG, "NULL id_out");
    static_assert(sizeof(ncclUniqueId) == RGNN_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    RGNN_NCCL(api().GetUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
  });
}

rgnn_status rgnn_comm_create(int32_t rank, int32_t world, const void* unique_id, const int64_t* node_ptr,
                             rgnn_comm_t* out) {
  return guarded([&] {
    RGNN_CHECK(out && unique_id && node_ptr, RGNN_ERR_INVALID_ARG, "NULL argument");
    RGNN_CHECK(world >= 1 && rank >= 0 && rank < world, RGNN_ERR_INVALID_ARG, "rank must lie in [0, world)");
    RGNN_CHECK(node_ptr[0] == 0, RGNN_ERR_INVALID_ARG, "node_ptr[0] must be 0");
    for (int k = 0; k < world; ++k)
      RGNN_CHECK(node_ptr[k + 1] >= node_ptr[k], RGNN_ERR_INVALID_ARG, "node_ptr must be non-decreasing");
    *out = nullptr;
    NcclApi& a = api();
    auto* c = new rgnn_comm_s();
    c->rank = rank;
    c->world = world;
    c->node_ptr.assign(node_ptr, node_ptr + world + 1);
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    try {
      RGNN_CUDA(cudaGetDevice(&c->device));
      RGNN_NCCL(a.CommInitRank(&c->nc, world, id, rank));
      int lo = 0, hi = 0;
      RGNN_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      RGNN_CUDA(cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, hi));
      c->chunk.resize(world);
      for (auto& e : c->chunk) RGNN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      RGNN_CUDA(cudaEventCreateWithFlags(&c->start, cudaEventDisableTiming));
      RGNN_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
    } catch (...) {
      rgnn_comm_destroy(c);
      throw;
    }
    *out = c;
  });
}

rgnn_status rgnn_comm_destroy(rgnn_comm_t c) {
  return guarded([&] {
    if (!c) return;
    if (c->cs) cudaStreamSynchronize(c->cs);
    for (auto e : c->chunk)
      if (e) cudaEventDestroy(e);
    if (c->start) cudaEventDestroy(c->start);
    if (c->done) cudaEventDestroy(c->done);
    if (c->cs) cudaStreamDestroy(c->cs);
    if (c->nc) api().CommDestroy(c->nc);
    delete c;
  });
}

rgnn_status rgnn_comm_info(rgnn_comm_t c, int32_t* rank, int32_t* world) {
  return guarded([&] {
    RGNN_CHECK(c, RGNN_ERR_INVALID_ARG, "NULL comm");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
  });
}

}  // extern "C"
