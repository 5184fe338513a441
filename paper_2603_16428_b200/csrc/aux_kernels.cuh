// aux_kernels.cuh — the small HBM-bound kernels around the GEMM core.
//   prep_targets      : n_valid and bad-target count (integer, bit-exact), resets the done counter.
//   local_combine     : merges the per-(row, vocab tile) (m, s) partials of one shard into the
//                       per-row ShardStat {m, s, z_t, hit}.
//   final_combine     : merges g ShardStats in shard order into lse, the per-row loss, the
//                       RowStat consumed by the backward, and the deterministic loss reduction.
#pragma once
#include <cstdint>

#include "../../include/slf_lce.h"
#include "ptx.cuh"

namespace slf {

struct WsHeader {
  unsigned long long n_valid;
  int bad;
  unsigned int done;
  unsigned long long pad[6];
};
constexpr size_t WS_HEADER_BYTES = 64 * 1024;  // header (256 B) + block partial sums (double) + sync area
// The header's last 8 KB: per-chunk synchronisation words of the in-kernel combine (schedule S,
// DESIGN.md §6): [chunk] {arrivals, fallback flag}, zeroed at the start of every call.
constexpr size_t WS_SYNC_BYTES = 8 * 1024;
constexpr size_t WS_SYNC_OFF = WS_HEADER_BYTES - WS_SYNC_BYTES;
constexpr int WS_SYNC_SLOTS = (int)(WS_SYNC_BYTES / 8);
// Blocks of 256 rows whose fp64 loss partials fit the header between its first 256 bytes and the
// sync area (7136 blocks: N <= 1,826,816 rows per statistics-combine call).
constexpr int MAX_LOSS_BLOCKS = (int)((WS_SYNC_OFF - 256) / 8);

// One block of 1024 threads: 16-byte vector loads of the targets.
__global__ void __launch_bounds__(1024) prep_targets_kernel(const int32_t* __restrict__ t, int64_t N,
                                                           int32_t ignore_index, int64_t V_global,
                                                           WsHeader* hdr) {
  unsigned long long nv = 0;
  int bad = 0;
  const int64_t n4 = N / 4;
  const int4* t4 = reinterpret_cast<const int4*>(t);
  auto acc = [&](int32_t x) {
    const bool valid = x != ignore_index;
    nv += valid;
    bad += (valid && (x < 0 || (int64_t)x >= V_global));
  };
  for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) {
    const int4 q = t4[i];
    acc(q.x); acc(q.y); acc(q.z); acc(q.w);
  }
  for (int64_t i = n4 * 4 + threadIdx.x; i < N; i += blockDim.x) acc(t[i]);
  for (int o = 16; o; o >>= 1) {
    nv += __shfl_xor_sync(0xffffffffu, nv, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ unsigned long long snv[32];
  __shared__ int sbad[32];
  if ((threadIdx.x & 31) == 0) { snv[threadIdx.x / 32] = nv; sbad[threadIdx.x / 32] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0;
    int b = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) { a += snv[w]; b += sbad[w]; }
    hdr->n_valid = a;
    hdr->bad = b;
    hdr->done = 0;
  }
}

// Thread = row: coalesced reads of partials[t * N + row] (stored [tile][row]).
__global__ void __launch_bounds__(256) local_combine_kernel(const float2* __restrict__ partials, int tiles,
                                                           const float* __restrict__ zt,
                                                           const int32_t* __restrict__ t, int64_t N,
                                                           int64_t vocab_start, int64_t V_local,
                                                           int32_t ignore_index, slf_shardstat* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  float m = -INFINITY, s = 0.f;
  for (int k = 0; k < tiles; ++k) {
    const float2 p = partials[(size_t)k * N + r];
    if (p.x > m) {
      s = s * ex2((m - p.x) * LOG2E) + p.y;
      m = p.x;
    } else {
      s += p.y * ex2((p.x - m) * LOG2E);
    }
  }
  const int32_t tt = t[r];
  const int64_t loc = (int64_t)tt - vocab_start;
  const bool hit = tt != ignore_index && loc >= 0 && loc < V_local;
  out[r] = slf_shardstat{m, s, hit ? zt[r] : 0.f, hit ? 1.f : 0.f};
}

// Thread = row.  g shard statistics in shard order -> lse, loss_i, RowStat; deterministic block
// partial sums (fixed tree) and a last-block final sum in fixed block order.
__global__ void __launch_bounds__(256) final_combine_kernel(const slf_shardstat* __restrict__ st, int g,
                                                           const int32_t* __restrict__ t, int64_t N,
                                                           int64_t vocab_start, int64_t V_local,
                                                           int64_t V_global, int32_t ignore_index, int reduction,
                                                           float scale, float* __restrict__ loss_out,
                                                           slf_rowstat* __restrict__ rowstat, WsHeader* hdr,
                                                           double* __restrict__ block_sums) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long n_valid = hdr->n_valid;
  const bool any_bad = hdr->bad > 0;
  double li = 0.0;
  if (r < N) {
    float M = -INFINITY;
    for (int k = 0; k < g; ++k) M = fmaxf(M, st[(size_t)k * N + r].m);
    float S = 0.f, z = 0.f;
    for (int k = 0; k < g; ++k) {
      const slf_shardstat q = st[(size_t)k * N + r];
      S += q.s * ex2((q.m - M) * LOG2E);
      z += q.zt;  // exactly one shard has hit = 1 (others store 0)
    }
    const float lse = M + logf(S);
    const int32_t tt = t[r];
    const bool valid = tt != ignore_index;
    const bool bad = valid && (tt < 0 || (int64_t)tt >= V_global);
    float l = valid ? (lse - z) : 0.f;
    if (bad) l = __int_as_float(0x7fc00000);
    float coef = 0.f;
    if (valid) coef = (reduction == SLF_MEAN) ? (n_valid ? scale / (float)n_valid : 0.f) : scale;
    const int64_t loc = (int64_t)tt - vocab_start;
    const int32_t tloc = (valid && !bad && loc >= 0 && loc < V_local) ? (int32_t)loc : -1;
    rowstat[r] = slf_rowstat{lse * LOG2E, bad ? 0.f : coef, tloc, valid ? 1 : 0};
    if (reduction == SLF_NONE) loss_out[r] = l;
    li = (double)l;
  }
  if (reduction == SLF_NONE) return;
  // Fixed-order block reduction.
  __shared__ double sh[256];
  sh[threadIdx.x] = li;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  __shared__ bool last;
  if (threadIdx.x == 0) {
    block_sums[blockIdx.x] = sh[0];
    __threadfence();
    const unsigned int prev = atomicAdd(&hdr->done, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Last block: sum the block partials in block order (each thread a fixed strided subset, then a
  // fixed tree), so the result does not depend on block scheduling.
  double a = 0.0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) a += ((volatile double*)block_sums)[b];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double tot = sh[0];
    if (reduction == SLF_MEAN) tot = n_valid ? tot / (double)n_valid : 0.0;
    loss_out[0] = any_bad ? __int_as_float(0x7fc00000) : (float)tot;
  }
}

// dhidden bf16 = RNE(fp32 sum of shard partials); ignored rows -> +0.0.  8 elements per thread.
__global__ void __launch_bounds__(256) dx_finalize_kernel(const float* __restrict__ in,
                                                         const slf_rowstat* __restrict__ rs, uint16_t* __restrict__ out,
                                                         int64_t N, int64_t H) {
  const int64_t groups = N * H / 8;
  for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = gi * 8 / H;
    const float4 a = reinterpret_cast<const float4*>(in)[2 * gi];
    const float4 b = reinterpret_cast<const float4*>(in)[2 * gi + 1];
    uint4 o = make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
    if (!rs[row].valid) o = make_uint4(0u, 0u, 0u, 0u);
    reinterpret_cast<uint4*>(out)[gi] = o;
  }
}

}  // namespace slf
