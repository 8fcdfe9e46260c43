// comm.cu — the multi-GPU step inside the library: an NCCL communicator per
// context and the whole sharded FMM step behind one call, so a C++ host runs it
// without torch. NCCL is bound at run time (dlopen of libnccl.so.2: the process's copy if one is
// already loaded, e.g. torch's), so single-GPU users never need it.
//
// fmm_evaluate_sharded, per rank (one process per GPU, every rank holds all bodies):
//   FMM stream    build (replicated) -> traversal (first step: full lists + cost plan; later steps:
//                 targets filtered to the rank's Morton range) -> P2P of the own leaves
//   comm stream   (after the traversal) P2M/M2M of the own cells -> pack -> ncclAllGather of the
//                 owned multipoles over NVLink -> unpack + shared ancestors
//   FMM stream    (joins the comm stream) M2L for targets meeting the range -> L2L -> L2P
// The all-gather, the step's only data-path exchange, runs under the P2P kernel.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "context.cuh"

namespace fmmb {
namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  std::string why;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) {
      api.why = "NCCL not found (dlopen libnccl.so.2)";
      return;
    }
    auto sym = [&](const char* n) { return dlsym(api.handle, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy)
      api.why = "NCCL library lacks the required entry points";
  });
  if (!api.why.empty()) fail(FMM_ERR_UNSUPPORTED, api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* s = nccl().error_string ? nccl().error_string(r) : "?";
  fail(FMM_ERR_CUDA, std::string("NCCL ") + what + ": " + s);
}

}  // namespace

void comm_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == FMM_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

int comm_version() {
  int v = 0;
  if (nccl().get_version) nccl().get_version(&v);
  return v;
}

void comm_init(fmm_ctx* c, const void* id128, int rank, int world) {
  comm_destroy(c);
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm = nullptr;
  nccl_check(nccl().comm_init_rank(&comm, world, id, rank), "ncclCommInitRank");
  c->nccl_comm = comm;
  c->comm_rank = rank;
  c->comm_world = world;
}

void comm_destroy(fmm_ctx* c) {
  if (c->nccl_comm) {
    nccl().comm_destroy(static_cast<ncclComm_t>(c->nccl_comm));
    c->nccl_comm = nullptr;
  }
  c->comm_rank = 0;
  c->comm_world = 0;
}

void comm_all_gather(fmm_ctx* c, const double* send, double* recv, size_t count, cudaStream_t s) {
  if (c->ag_fn) {
    if (c->ag_fn(send, recv, static_cast<int64_t>(count), s, c->ag_user) != 0)
      fail(FMM_ERR_CUDA, "all-gather callback failed");
    return;
  }
  if (!c->nccl_comm) fail(FMM_ERR_STATE, "no communicator (fmm_comm_init)");
  nccl_check(nccl().all_gather(send, recv, count, ncclFloat64, static_cast<ncclComm_t>(c->nccl_comm), s),
             "ncclAllGather");
}

}  // namespace fmmb
