// nccl_hook.cpp — native NCCL all-reduce for the K-Means Lloyd loop's
// per-iteration centroid partials (hpac_kmeans_problem_t.allreduce), so a C++
// driver shards points across the GPUs of a node without Python:
//
//   ncclComm_t comm;  ncclCommInitRank(&comm, nranks, id, rank);   // caller's
//   pb.allreduce = hpac_nccl_allreduce;  pb.allreduce_user = comm;
//   hpac_kmeans_run(&grid, &pb, spec, stream, &res, err, sizeof err);
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): the library keeps no
// link-time NCCL dependency and shares whichever libnccl the process already
// loaded (e.g. the one torch ships). ncclAllReduce(sum, double) in place on
// the caller's stream, over NVLink/NVSwitch within a node.
#include <dlfcn.h>

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "hpac_offload.h"

#define HPAC_API extern "C" __attribute__((visibility("default")))

namespace {
typedef int (*AllReduceFn)(const void*, void*, size_t, int /*dtype*/, int /*op*/, void* /*comm*/,
                           void* /*stream*/);
typedef int (*InitAllFn)(void** /*comms*/, int, const int*);
typedef int (*DestroyFn)(void*);
typedef int (*AsyncErrFn)(void*, int*);
struct NcclUid {  // nccl.h ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128)
  char internal[128];
};
typedef int (*GetUidFn)(NcclUid*);
typedef int (*InitRankFn)(void** /*comm*/, int /*nranks*/, NcclUid /*id, by value*/, int /*rank*/);
constexpr int kNcclFloat64 = 8, kNcclSum = 0;  // nccl.h ncclDataType_t / ncclRedOp_t

struct Nccl {
  void* h = nullptr;
  AllReduceFn all_reduce = nullptr;
  InitAllFn init_all = nullptr;
  DestroyFn destroy = nullptr;
  GetUidFn get_uid = nullptr;
  InitRankFn init_rank = nullptr;
  AsyncErrFn async_err = nullptr;
};

Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) return;
    n.all_reduce = reinterpret_cast<AllReduceFn>(dlsym(n.h, "ncclAllReduce"));
    n.init_all = reinterpret_cast<InitAllFn>(dlsym(n.h, "ncclCommInitAll"));
    n.destroy = reinterpret_cast<DestroyFn>(dlsym(n.h, "ncclCommDestroy"));
    n.get_uid = reinterpret_cast<GetUidFn>(dlsym(n.h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<InitRankFn>(dlsym(n.h, "ncclCommInitRank"));
    n.async_err = reinterpret_cast<AsyncErrFn>(dlsym(n.h, "ncclCommGetAsyncError"));
  });
  return n.all_reduce ? &n : nullptr;
}
}  // namespace

HPAC_API int hpac_nccl_available(void) { return nccl() != nullptr; }

// hpac_allreduce_fn: `user` is the caller's ncclComm_t. A missing NCCL or
// communicator and a failing ncclAllReduce are reported, never skipped: the
// Lloyd loop then stops with HPAC_ERR_CUDA instead of continuing on this
// rank's un-reduced partials.
HPAC_API int hpac_nccl_allreduce(double* buf, int64_t count, void* user, void* stream) {
  Nccl* n = nccl();
  if (!n || !user) return HPAC_ERR_UNSUPPORTED;
  return n->all_reduce(buf, buf, (size_t)count, kNcclFloat64, kNcclSum, user, stream) == 0
             ? HPAC_OK
             : HPAC_ERR_CUDA;
}

// Asynchronous communicator errors (ncclCommGetAsyncError): a collective
// that failed after it was enqueued (e.g. inside a graph launch).
HPAC_API int hpac_nccl_check(void* comm) {
  Nccl* n = nccl();
  if (!n || !comm) return HPAC_ERR_UNSUPPORTED;
  if (!n->async_err) return HPAC_OK;
  int state = 0;  // ncclSuccess
  if (n->async_err(comm, &state) != 0) return HPAC_ERR_CUDA;
  return state == 0 || state == 7 /* ncclInProgress */ ? HPAC_OK : HPAC_ERR_CUDA;
}

// Single-process communicators over `ndev` local devices (ncclCommInitAll),
// for drivers and tests that own every GPU of the node in one process.
HPAC_API int hpac_nccl_comm_init_all(int ndev, const int* devlist, void** comms) {
  Nccl* n = nccl();
  if (!n || !n->init_all) return HPAC_ERR_UNSUPPORTED;
  return n->init_all(comms, ndev, devlist) == 0 ? HPAC_OK : HPAC_ERR_CUDA;
}

// Multi-process communicators (one process per GPU, e.g. under torchrun):
// rank 0 creates the 128-byte id, the caller broadcasts it (any channel),
// every rank then joins. With this communicator as the hook's `user`, the
// Lloyd loop's all-reduce is captured into its CUDA graph.
HPAC_API int hpac_nccl_unique_id(uint8_t* id128) {
  Nccl* n = nccl();
  if (!n || !n->get_uid || !id128) return HPAC_ERR_UNSUPPORTED;
  NcclUid id;
  if (n->get_uid(&id) != 0) return HPAC_ERR_CUDA;
  std::memcpy(id128, id.internal, sizeof id.internal);
  return HPAC_OK;
}

HPAC_API int hpac_nccl_comm_init_rank(int nranks, const uint8_t* id128, int rank, void** comm) {
  Nccl* n = nccl();
  if (!n || !n->init_rank || !id128 || !comm) return HPAC_ERR_UNSUPPORTED;
  NcclUid id;
  std::memcpy(id.internal, id128, sizeof id.internal);
  return n->init_rank(comm, nranks, id, rank) == 0 ? HPAC_OK : HPAC_ERR_CUDA;
}

HPAC_API int hpac_nccl_comm_destroy(void* comm) {
  Nccl* n = nccl();
  if (!n || !n->destroy) return HPAC_ERR_UNSUPPORTED;
  return n->destroy(comm) == 0 ? HPAC_OK : HPAC_ERR_CUDA;
}
