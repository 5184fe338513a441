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

// ---- P2P one-shot all-gather of the per-chunk statistics ----------------
// Every rank owns a receive buffer [flags | 2 parities x world x C x 16 B] in its own device memory,
// mapped into every peer through CUDA IPC.  Chunk e (a communicator-wide epoch, 1, 2, ...): each rank
// stores its C x 16 B statistics straight into slot `rank` of parity e % 2 of EVERY rank's buffer
// (NVLink stores; one block per destination), then, after a system-scope fence, adds 1 to its own
// counter flags[rank] in each destination (release).  A rank's chunk-e consumer waits until all g
// counters of its own buffer reach e (acquire), then reads the g slots locally.  Two parities
// suffice: a peer can only write epoch e+2 after it has seen this rank's epoch e+1 statistics, which
// this rank pushes after its epoch-e consumer has finished (stream order).
constexpr int P2P_MAX_RANKS = 16;
constexpr size_t P2P_HDR_BYTES = 256;  // flags[P2P_MAX_RANKS] u64 + error word at byte 192
struct PeerPtrs {
  uint8_t* p[P2P_MAX_RANKS];
};

__global__ void __launch_bounds__(256) p2p_stats_push_kernel(const uint4* __restrict__ st, int rows, int rank,
                                                             PeerPtrs peers, size_t data_off) {
  uint8_t* base = peers.p[blockIdx.x];
  uint4* dst = reinterpret_cast<uint4*>(base + data_off) + (size_t)rank * rows;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) dst[i] = st[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* flag = reinterpret_cast<unsigned long long*>(base) + rank;
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(flag) : "memory");
  }
}

// Thread r < g waits for flags[r] >= target (bounded: ~30 s, then the error word is set and the
// consumer reads whatever is there — slf_comm_status reports it; no hang).
__global__ void p2p_stats_wait_kernel(uint8_t* buf, int g, unsigned long long target) {
  const int r = threadIdx.x;
  if (r >= g) return;
  const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(buf) + r;
  for (long long spins = 0;; ++spins) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    if (spins > (1ll << 27)) {
      atomicExch(reinterpret_cast<int*>(buf + 192), 1);
      break;
    }
    __nanosleep(200);
  }
}

}  // namespace slf

// The handle behind slf_comm (opaque in the header).
struct slf_comm_s {
  int rank = 0, world = 1, device = 0;
  // NCCL transport
  ncclComm_t nccl = nullptr;
  cudaStream_t cs = nullptr;  // the communicator's stream
  cudaEvent_t ev_in = nullptr, ev_ag = nullptr, ev_ar[2] = {nullptr, nullptr};
  // P2P statistics all-gather (slf_comm_set_p2p)
  bool p2p = false;
  uint8_t* p2p_buf = nullptr;  // this rank's receive buffer (cudaMalloc, communicator-owned)
  int64_t p2p_rows = 0;        // capacity in rows per slot
  uint8_t* p2p_peer[slf::P2P_MAX_RANKS] = {};  // mapped receive buffers of every rank (own = p2p_buf)
  unsigned long long epoch = 0;
  // callback transport
  slf_allgather_fn cb_allgather = nullptr;
  slf_allreduce_f32_fn cb_allreduce = nullptr;
  void* cb_user = nullptr;
};
