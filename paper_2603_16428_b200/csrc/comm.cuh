// comm.cuh — the collective transport of the vocab-sharded path (SURVEY §8(b) "Comm", §8(e)).
//
// Two transports behind one handle (slf_comm):
//   * NCCL, loaded at run time with dlopen("libnccl.so.2") — the copy PyTorch already loaded when
//     there is one (RTLD_NOLOAD first), else the system library.  The library itself links no NCCL,
//     so it loads on machines without one; slf_comm_init then fails with SLF_ERR_COMM.
//     Every collective of a communicator runs on ONE internal stream (`cs`), in issue order, as
//     PyTorch's ProcessGroupNCCL does: the caller's stream and the comm stream are joined by events,
//     so the fp32 dX all-reduce of chunk c overlaps the stash GEMM of chunk c+1.
//   * caller callbacks (tests: e.g. gloo through host copies, two processes on one GPU), invoked
//     synchronously on the calling thread.
// Only the types of nccl.h are used here; every function comes from the dlopen'ed library.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "../../include/slf_lce.h"

namespace slf {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  char why[256] = {0};
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(api.why, sizeof(api.why), "cannot load libnccl.so.2: %s", dlerror());
      return;
    }
    bool all = true;
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp) {
        all = false;
        snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks %s", name);
      }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllGather, "ncclAllGather");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = all;
  });
  return api;
}

}  // namespace slf

// The handle behind slf_comm (opaque in the header).
struct slf_comm_s {
  int rank = 0, world = 1, device = 0;
  // NCCL transport
  ncclComm_t nccl = nullptr;
  cudaStream_t cs = nullptr;  // the communicator's stream
  cudaEvent_t ev_in = nullptr, ev_ag = nullptr, ev_ar[2] = {nullptr, nullptr};
  // callback transport
  slf_allgather_fn cb_allgather = nullptr;
  slf_allreduce_f32_fn cb_allreduce = nullptr;
  void* cb_user = nullptr;
};
