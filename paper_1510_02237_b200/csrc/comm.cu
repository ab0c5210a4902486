// Collectives of the row-sharded sweep, enqueued from C++ on the context
// stream: the serial correction's allreduce of the partial alpha_{i+1} (r doubles) and
// all-gather of qn_{i+1}'s row blocks, and the TSQR all-gather of the R factors
// (reference serial loop parareal.py:128-132; subspace.py:60-74).
//
// Two transports behind one interface:
//  * NCCL (pw_ctx_set_nccl): the library owns an ncclComm_t built from a unique id the
//    host side broadcasts once (torch.distributed in dist.NcclComm).  No host round-trip
//    per serial step: the calls are stream-ordered like the kernels around them.  NCCL
//    is resolved at run time (dlopen of libnccl.so.2 -- RTLD_NOLOAD first, so a process
//    that already loaded torch's NCCL uses that one), so the library has no link-time
//    NCCL dependency and single-GPU use never touches it.
//  * the ctypes hooks of pw_ctx_set_comm (gloo tests, thread ranks).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "pw_internal.h"

namespace pw {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.allGather &&
             api.getErrorString;
  });
  PW_CHECK(api.ok, PW_ERR_STATE, "NCCL (libnccl.so.2) is not available in this process");
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error{PW_ERR_STATE, std::string(what) + ": " + nccl().getErrorString(r)};
}

}  // namespace

void nccl_unique_id(unsigned char* out) {
  ncclUniqueId id;
  check(nccl().getUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "NCCL unique ids are 128 bytes");
  memcpy(out, &id, sizeof(id));
}

void nccl_init(Ctx& c, const unsigned char* id_bytes, int rank, int world) {
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof(id));
  PW_CUDA(cudaSetDevice(c.device));
  ncclComm_t comm = nullptr;
  check(nccl().commInitRank(&comm, world, id, rank), "ncclCommInitRank");
  if (c.nccl) nccl().commDestroy(static_cast<ncclComm_t>(c.nccl));
  c.nccl = comm;
  c.comm_rank = rank;
  c.comm_world = world;
}

void nccl_destroy(Ctx& c) {
  if (c.nccl) {
    nccl().commDestroy(static_cast<ncclComm_t>(c.nccl));
    c.nccl = nullptr;
  }
}

// in-place sum over ranks of count doubles (stream-ordered)
void comm_allreduce(Ctx& c, double* data, long long count) {
  if (c.nccl) {
    check(nccl().allReduce(data, data, (size_t)count, ncclDouble, ncclSum, static_cast<ncclComm_t>(c.nccl),
                           c.stream),
          "ncclAllReduce");
    return;
  }
  PW_CHECK(c.allreduce_hook && c.allreduce_hook(c.comm_user, data, count) == 0, PW_ERR_STATE,
           "allreduce hook failed");
}

// data[rank*block .. +block) valid on this rank (the last block may be short): fill the
// others.  NCCL needs equal, padded blocks: through a world x block scratch buffer.
void comm_allgather(Ctx& c, double* data, long long block, long long total) {
  PW_CHECK(total <= (long long)c.comm_world * block, PW_ERR_VALUE, "all-gather blocks do not cover the vector");
  if (c.nccl) {
    const size_t need = (size_t)c.comm_world * (size_t)block;
    if (c.comm_scratch_n < need) {
      if (c.comm_scratch) PW_CUDA(cudaFreeAsync(c.comm_scratch, c.stream));
      PW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c.comm_scratch), need * sizeof(double), c.stream));
      PW_CUDA(cudaMemsetAsync(c.comm_scratch, 0, need * sizeof(double), c.stream));
      c.comm_scratch_n = need;
    }
    const long long lo = std::min<long long>(total, (long long)c.comm_rank * block);
    const long long hi = std::min<long long>(total, lo + block);
    double* mine = c.comm_scratch + (size_t)c.comm_rank * block;
    if (hi > lo)
      PW_CUDA(cudaMemcpyAsync(mine, data + lo, sizeof(double) * (hi - lo), cudaMemcpyDeviceToDevice, c.stream));
    check(nccl().allGather(mine, c.comm_scratch, (size_t)block, ncclDouble, static_cast<ncclComm_t>(c.nccl),
                           c.stream),
          "ncclAllGather");
    PW_CUDA(cudaMemcpyAsync(data, c.comm_scratch, sizeof(double) * total, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  PW_CHECK(c.allgather_hook && c.allgather_hook(c.comm_user, data, block, total) == 0, PW_ERR_STATE,
           "all-gather hook failed");
}

}  // namespace pw
