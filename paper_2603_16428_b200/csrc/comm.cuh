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
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/slf_lce.h"
#include "ptx.cuh"

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
// Header of a rank's receive buffer: statistics counters [16] u64 at 0, the timeout word at 192,
// dX "partial ready" counters [16] u64 at 256, dX "slice delivered" counters [16] u64 at 384, the
// exchange kernel's finished-block counter (u32) at 512.
constexpr size_t P2P_HDR_BYTES = 1024;
constexpr size_t P2P_ERR_OFF = 192, P2P_DX_READY_OFF = 256, P2P_DX_DONE_OFF = 384, P2P_DX_BLOCKS_OFF = 512;
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
// consumer reads whatever is there — slf_comm_status reports it; no hang).  `off`: which counters.
__global__ void p2p_stats_wait_kernel(uint8_t* buf, int g, unsigned long long target, int off = 0) {
  const int r = threadIdx.x;
  if (r >= g) return;
  const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(buf + off) + r;
  for (long long spins = 0;; ++spins) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    if (spins > (1ll << 27)) {
      atomicExch(reinterpret_cast<int*>(buf + P2P_ERR_OFF), 1);
      break;
    }
    __nanosleep(200);
  }
}

__device__ __forceinline__ void p2p_spin_geq(const unsigned long long* flag, unsigned long long target, uint8_t* buf) {
  for (long long spins = 0;; ++spins) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) return;
    if (spins > (1ll << 27)) {
      atomicExch(reinterpret_cast<int*>(buf + P2P_ERR_OFF), 1);
      return;
    }
    __nanosleep(200);
  }
}

// The dX exchange of one chunk as one kernel (NEXT-3 / DESIGN.md §9b): on rank k, after this
// rank's fp32 partial of the chunk is complete, (a) announce it to every rank, (b) wait until every
// rank's partial is there, (c) for the rows of this rank's slice [s0, s1) of the chunk, sum the g
// partials in rank order (deterministic; peer memory over NVLink), round to bf16 (ignored rows +0)
// and store the rows into EVERY rank's dhidden (the all-gather), (d) the last block to finish tells
// every rank that its partial has been read and its dhidden slice written.  Reduce-scatter +
// all-gather + finalize in one pass, no NCCL; it runs on the comm stream on the SMs the GEMMs
// leave free, under the next chunk's stash GEMM.
struct DxArgs {
  PeerPtrs part;   // each rank's fp32 partial of this chunk, row 0 ([rows][H])
  PeerPtrs dx;     // each rank's dhidden at the chunk's row 0 (bf16 [rows][H])
  PeerPtrs flags;  // each rank's receive buffer (header)
  const slf_rowstat* rowstat;  // this chunk's row 0
  uint8_t* mybuf;
  int g, rank, s0, s1, H;
  unsigned long long epoch;
};

__global__ void __launch_bounds__(256) p2p_dx_exchange_kernel(DxArgs a) {
  if (blockIdx.x == 0 && threadIdx.x < a.g) {  // (a) my partial of this epoch is ready
    unsigned long long* f = reinterpret_cast<unsigned long long*>(a.flags.p[threadIdx.x] + P2P_DX_READY_OFF) + a.rank;
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(f) : "memory");
  }
  if (threadIdx.x < a.g)  // (b)
    p2p_spin_geq(reinterpret_cast<const unsigned long long*>(a.mybuf + P2P_DX_READY_OFF) + threadIdx.x, a.epoch,
                 a.mybuf);
  __syncthreads();
  // (c) 8 columns (two 16-byte fp32 loads per rank, one 16-byte bf16 store per rank) per item
  const int per_row = a.H / 8;
  const long long items = (long long)(a.s1 - a.s0) * per_row;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int r = a.s0 + (int)(it / per_row);
    const int c = (int)(it % per_row) * 8;
    float acc[8];
    {
      const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.part.p[0]) +
                                                          (size_t)r * a.H + c);
      const float4 x0 = src[0], x1 = src[1];
      acc[0] = x0.x; acc[1] = x0.y; acc[2] = x0.z; acc[3] = x0.w;
      acc[4] = x1.x; acc[5] = x1.y; acc[6] = x1.z; acc[7] = x1.w;
    }
#pragma unroll 4
    for (int p = 1; p < a.g; ++p) {  // rank order (unrolled: the peers' loads are in flight together)
      const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.part.p[p]) +
                                                          (size_t)r * a.H + c);
      const float4 x0 = src[0], x1 = src[1];
      acc[0] += x0.x; acc[1] += x0.y; acc[2] += x0.z; acc[3] += x0.w;
      acc[4] += x1.x; acc[5] += x1.y; acc[6] += x1.z; acc[7] += x1.w;
    }
    uint4 o = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                         pack_bf16x2(acc[6], acc[7]));
    if (!a.rowstat[r].valid) o = make_uint4(0u, 0u, 0u, 0u);
    for (int p = 0; p < a.g; ++p)
      *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.dx.p[p]) + (size_t)r * a.H + c) = o;
  }
  // (d) every store of this block is visible system-wide before the block counts itself done
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int* cnt = reinterpret_cast<unsigned int*>(a.mybuf + P2P_DX_BLOCKS_OFF);
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
      *cnt = 0u;  // the next chunk's kernel runs after this one (same stream)
      __threadfence_system();
      for (int p = 0; p < a.g; ++p) {
        unsigned long long* f = reinterpret_cast<unsigned long long*>(a.flags.p[p] + P2P_DX_DONE_OFF) + a.rank;
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(f) : "memory");
      }
    }
  }
}

// After a sharded step with P2P exchanges: if any wait of this rank timed out (error word set), the
// step's results are invalid — poison the loss with NaN (the ABI's asynchronous data-error
// convention, as for bad targets) and raise the host-mapped sticky flag that makes the next
// slf_lce_fwd_bwd_sharded call on this communicator return SLF_ERR_COMM.
__global__ void p2p_check_kernel(const uint8_t* buf, float* loss, int64_t n_loss, volatile int* host_flag) {
  if (*reinterpret_cast<const volatile int*>(buf + P2P_ERR_OFF) == 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_loss; i += (int64_t)gridDim.x * blockDim.x)
    loss[i] = __int_as_float(0x7fc00000);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *host_flag = 1;
    __threadfence_system();
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
  // P2P exchanges (slf_comm_set_p2p): bit 0 statistics all-gather, bit 1 dX exchange kernel
  bool p2p = false;
  int p2p_mode = 0;
  uint8_t* p2p_buf = nullptr;  // this rank's receive buffer (cudaMalloc, communicator-owned)
  int64_t p2p_rows = 0;        // capacity in rows per slot
  uint8_t* p2p_peer[slf::P2P_MAX_RANKS] = {};  // mapped receive buffers of every rank (own = p2p_buf)
  int* p2p_err_host = nullptr;  // sticky timeout flag, pinned host memory mapped into the device
  int* p2p_err_dev = nullptr;   // its device alias
  unsigned long long epoch = 0;
  unsigned long long dx_epoch = 0;  // chunks whose dX went through the exchange kernel
  // caller buffers mapped from peers: (handle bytes) -> opened base, and this rank's exported bases
  std::vector<std::pair<std::string, uint8_t*>> ipc_open;
  // callback transport
  slf_allgather_fn cb_allgather = nullptr;
  slf_allreduce_f32_fn cb_allreduce = nullptr;
  void* cb_user = nullptr;
};
