// s_kernels.cuh — HBM-bound kernels of schedule S (no recompute).
//   combine_transform : per row of a chunk: merge the (m_t, s_t) tile statistics into lse, the row
//                       loss and RowStat, then rescale the bf16 stash p~ = exp(z - m_t) in place
//                       into G_P = coef * exp(z - lse)  (softmax term only; the one-hot term is
//                       applied exactly elsewhere: dX epilogue and onehot_kernel).
//   csr_*             : stable counting sort of the valid in-shard tokens by target id (the
//                       "target CSR"): counts, exclusive scan + hit list, rank by brute force over
//                       earlier tokens (deterministic, no atomics on positions), scatter.
//   onehot_kernel     : dW[v] -= coef * sum_{i in CSR[v]} x_i, summed in fp32 in token order.
//   loss_reduce       : deterministic sum of the per-row losses.
#pragma once
#include <cstdint>

#include "../../include/slf_lce.h"
#include "aux_kernels.cuh"
#include "combine_dev.cuh"
#include "ptx.cuh"
#include "rmsnorm.cuh"

namespace slf {

// This shard's per-row ShardStat {m, s, z_t, hit} of a chunk: 8 rows per block of 256 threads, 32
// lanes per row; lane p merges tiles p, p+32, ... of the [tile][row] partials online (for a fixed
// tile the 8 rows' lanes read 8 consecutive partials, 64 bytes), then one thread per row merges the
// 32 lane results in lane order (fixed, deterministic).  Round 1 used four lanes per row over 32
// rows per block: fine for the ~63 tiles of a g = 8 shard, latency-bound for the 250-500 tiles of
// g <= 2 (41 us per 1024-row chunk at world 1).
constexpr int SR_ROWS = 8, SR_LANES = 32;
__global__ void __launch_bounds__(256) shard_rows_tpr_kernel(const float2* __restrict__ partials, int tiles, int rows,
                                                             const float* __restrict__ zt,
                                                             const int32_t* __restrict__ t, int64_t vocab_start,
                                                             int64_t V_l, int32_t ignore_index,
                                                             slf_shardstat* __restrict__ out) {
  __shared__ float lm[SR_LANES][SR_ROWS], ls[SR_LANES][SR_ROWS];
  const int rl = threadIdx.x % SR_ROWS, lane = threadIdx.x / SR_ROWS;
  const int i0 = blockIdx.x * SR_ROWS;
  {
    const int i = i0 + rl;
    float m = -INFINITY, sum = 0.f;
    if (i < rows) {
#pragma unroll 4
      for (int k = lane; k < tiles; k += SR_LANES) {
        const float2 p = partials[(size_t)k * rows + i];
        const float nm = fmaxf(m, p.x);
        sum = (m == -INFINITY ? 0.f : sum * ex2((m - nm) * LOG2E)) + p.y * ex2((p.x - nm) * LOG2E);
        m = nm;
      }
    }
    lm[lane][rl] = m;
    ls[lane][rl] = sum;
  }
  __syncthreads();
  if (threadIdx.x >= SR_ROWS || i0 + (int)threadIdx.x >= rows) return;
  const int r = threadIdx.x, i = i0 + r;
  float M = -INFINITY, S = 0.f;
  for (int p = 0; p < SR_LANES; ++p) M = fmaxf(M, lm[p][r]);
  for (int p = 0; p < SR_LANES; ++p)
    if (lm[p][r] != -INFINITY) S += ls[p][r] * ex2((lm[p][r] - M) * LOG2E);
  const int32_t tt = t[i];
  const int64_t loc = (int64_t)tt - vocab_start;
  const bool hit = tt != ignore_index && loc >= 0 && loc < V_l;
  out[i] = slf_shardstat{M, S, hit ? zt[i] : 0.f, hit ? 1.f : 0.f};
}

// One block (256 threads) per row of the chunk.  The row's global statistics come from the g
// shards' ShardStats (fixed shard order; g = 1 on one GPU), the per-tile rescale factors from this
// shard's own tile partials.  Deterministic.
__global__ void __launch_bounds__(256) combine_transform_kernel(
    const slf_shardstat* __restrict__ st, int g, const float2* __restrict__ partials, int tiles, int rows,
    const float* __restrict__ zt, const int32_t* __restrict__ t, int64_t vocab_start, int64_t V_l, int64_t V_global,
    int64_t ld_stash, int32_t ignore_index, int reduction, float scale, float grad_scale,
    const WsHeader* __restrict__ hdr, float* __restrict__ loss_rows, slf_rowstat* __restrict__ rowstat,
    uint16_t* __restrict__ stash, uint16_t* __restrict__ stash2, int split, RmsStep rms) {
  // rows [0, split) of the chunk's stash are in `stash`, rows [split, rows) in `stash2` (same stride)
  extern __shared__ float r_t[];  // [tiles]: first the tile maxima m_t, then the factors r_t
  griddep_launch_dependents();
  griddep_wait();  // PDL: everything below reads the previous kernel's outputs
  if ((int)blockIdx.x >= rows) {  // the fused final RMSNorm's jobs riding in this launch (rmsnorm.cuh)
    rms_block(rms, (int64_t)blockIdx.x - rows);
    return;
  }
  __shared__ float sM, sLse, wm[8], ws[8];
  const int i = blockIdx.x;
  const int tid = threadIdx.x;
  uint4* row = reinterpret_cast<uint4*>(i < split ? stash + (size_t)i * ld_stash : stash2 + (size_t)(i - split) * ld_stash);
  const int64_t groups = (V_l + 7) / 8;
  constexpr int U = 8;  // 8 independent 16-byte loads in flight per thread (4: 1.94 ms, 16: no gain)
  // The first batch of the row is requested before the statistics are merged (latency overlap).
  uint4 w[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (tid + u * 256 < groups) w[u] = row[tid + u * 256];
  // One pass over this shard's tile partials: keep m_t in smem, merge (m, s) online per thread,
  // then a fixed-order warp-shuffle tree and a fixed-order pass over the 8 warps (deterministic).
  float m = -INFINITY, sum = 0.f;
  for (int k = tid; k < tiles; k += 256) {
    const float2 p = partials[(size_t)k * rows + i];
    r_t[k] = p.x;
    if (st == nullptr) {
      const float nm = fmaxf(m, p.x);
      sum = sum * ex2((m - nm) * LOG2E) + p.y * ex2((p.x - nm) * LOG2E);
      m = nm;
    }
  }
  if (st == nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_down_sync(0xffffffffu, m, o), os = __shfl_down_sync(0xffffffffu, sum, o);
      const float nm = fmaxf(m, om);
      sum = (m == -INFINITY ? 0.f : sum * ex2((m - nm) * LOG2E)) + (om == -INFINITY ? 0.f : os * ex2((om - nm) * LOG2E));
      m = nm;
    }
    if ((tid & 31) == 0) {
      wm[tid >> 5] = m;
      ws[tid >> 5] = sum;
    }
  }
  __syncthreads();
  if (tid == 0) {
    float M = -INFINITY, S = 0.f, z = 0.f;
    const int32_t tt = t[i];
    if (st == nullptr) {  // one GPU: this shard's own tiles
      for (int k = 0; k < 8; ++k) M = fmaxf(M, wm[k]);
      for (int k = 0; k < 8; ++k)
        if (wm[k] != -INFINITY) S += ws[k] * ex2((wm[k] - M) * LOG2E);
      const int64_t loc0 = (int64_t)tt - vocab_start;
      if (tt != ignore_index && loc0 >= 0 && loc0 < V_l) z = zt[i];
    } else {
      for (int k = 0; k < g; ++k) M = fmaxf(M, st[(size_t)k * rows + i].m);
      for (int k = 0; k < g; ++k) {
        const slf_shardstat q = st[(size_t)k * rows + i];
        S += q.s * ex2((q.m - M) * LOG2E);
        z += q.zt;  // exactly one shard has the target (the others store 0)
      }
    }
    const float lse = M + logf(S);
    const bool valid = tt != ignore_index;
    const bool bad = valid && (tt < 0 || (int64_t)tt >= V_global);
    const float coef = (valid && !bad) ? coef_of(reduction, scale, hdr->n_valid) : 0.f;
    float l = valid ? (lse - z) : 0.f;
    if (bad) l = __int_as_float(0x7fc00000);
    loss_rows[i] = l;
    const int64_t loc = (int64_t)tt - vocab_start;
    const int32_t tloc = (valid && !bad && loc >= 0 && loc < V_l) ? (int32_t)loc : -1;
    rowstat[i] = slf_rowstat{lse * LOG2E, coef, tloc, valid ? 1 : 0};
    sM = coef * grad_scale;
    sLse = lse * LOG2E;
  }
  __syncthreads();
  const float cg = sM, lse2 = sLse;
  for (int k = tid; k < tiles; k += 256) r_t[k] = cg * ex2(r_t[k] * LOG2E - lse2);
  __syncthreads();
  // G_P = p~ * r_t, in place, 8 bf16 per 16-byte access.
  for (int64_t q0 = tid;;) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * 256;
      if (q < groups) {
        const float r = r_t[(q * 8) / 256];
        uint4 x = w[u];
        x.x = pack_bf16x2(bf16lo_to_f32(x.x) * r, bf16hi_to_f32(x.x) * r);
        x.y = pack_bf16x2(bf16lo_to_f32(x.y) * r, bf16hi_to_f32(x.y) * r);
        x.z = pack_bf16x2(bf16lo_to_f32(x.z) * r, bf16hi_to_f32(x.z) * r);
        x.w = pack_bf16x2(bf16lo_to_f32(x.w) * r, bf16hi_to_f32(x.w) * r);
        row[q] = x;
      }
    }
    q0 += 256 * U;
    if (q0 >= groups) break;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q0 + u * 256 < groups) w[u] = row[q0 + u * 256];
  }
}

// ---- per-row stash reference ----------------------------------------------------
// The stash GEMM can store p~ = exp(z - M_i) against a per-row reference M_i fixed BEFORE the GEMM
// instead of each tile's own max; then G_P = coef * exp(z - lse) = p~ * f_i with one factor per row,
// f_i = coef * exp(M_i - lse_i), which the grouped GEMMs apply without touching the stash: dX's
// epilogue multiplies the row's accumulator by f_i, and dW's B operand is X'_chunk = bf16(f ⊙ X).
// M_i = z_{i,t_i} + STASH_REF_SHIFT (the target logit, a dot product per row): the row max is then at
// most M_i + 88 unless the target's loss exceeds ~128 nats, and entries below M_i - 87 (lost to
// underflow) have softmax < e^-47.  Rows that are ignored or whose target is out of range get
// M_i = +inf: their stash row is exactly 0 (and coef = 0).
constexpr float STASH_REF_SHIFT = 40.f;

// One warp per row: M_i = x_i . W[t_i - vocab_start] + STASH_REF_SHIFT (fp32, 16-byte loads).
// partial = 1 (vocab shards): this shard's target-logit contribution (0 for targets elsewhere), to be
// summed across shards and finished by mref_finish_kernel.
__global__ void __launch_bounds__(256) mref_kernel(const uint16_t* __restrict__ X, const uint16_t* __restrict__ W,
                                                  const int32_t* __restrict__ t, int64_t N, int64_t H,
                                                  int32_t ignore_index, int64_t vocab_start, int64_t V_l,
                                                  float* __restrict__ mref, int partial = 0) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= N) return;
  const int32_t tt = t[row];
  const int64_t loc = (int64_t)tt - vocab_start;
  if (tt == ignore_index || loc < 0 || loc >= V_l) {
    if (lane == 0) mref[row] = partial ? 0.f : INFINITY;
    return;
  }
  const uint4* xr = reinterpret_cast<const uint4*>(X + row * H);
  const uint4* wr = reinterpret_cast<const uint4*>(W + loc * H);
  float acc = 0.f;
  for (int64_t q = lane; q < H / 8; q += 32) {
    const uint4 a = xr[q], b = wr[q];
    acc = fmaf(bf16lo_to_f32(a.x), bf16lo_to_f32(b.x), acc); acc = fmaf(bf16hi_to_f32(a.x), bf16hi_to_f32(b.x), acc);
    acc = fmaf(bf16lo_to_f32(a.y), bf16lo_to_f32(b.y), acc); acc = fmaf(bf16hi_to_f32(a.y), bf16hi_to_f32(b.y), acc);
    acc = fmaf(bf16lo_to_f32(a.z), bf16lo_to_f32(b.z), acc); acc = fmaf(bf16hi_to_f32(a.z), bf16hi_to_f32(b.z), acc);
    acc = fmaf(bf16lo_to_f32(a.w), bf16lo_to_f32(b.w), acc); acc = fmaf(bf16hi_to_f32(a.w), bf16hi_to_f32(b.w), acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) mref[row] = partial ? acc : acc + STASH_REF_SHIFT;
}

// After the cross-shard sum of the partial target logits: M_i = z_t + shift, or +inf for ignored
// rows and targets outside [0, V_global).
__global__ void __launch_bounds__(256) mref_finish_kernel(const int32_t* __restrict__ t, int64_t N,
                                                         int32_t ignore_index, int64_t V_global,
                                                         float* __restrict__ mref) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int32_t tt = t[i];
  mref[i] = (tt == ignore_index || tt < 0 || (int64_t)tt >= V_global) ? INFINITY : mref[i] + STASH_REF_SHIFT;
}

// CS_ROWS = 8 rows per block of 256 threads (single GPU): each row's lse / loss / RowStat from its
// tile partials — 32 lanes per row merge interleaved tiles (lane p: tiles p, p+32, ...; for a fixed
// tile the 8 rows' lanes read 8 consecutive partials, two 32-byte sectors), then one thread per row
// merges the 32 lane results in lane order (fixed, deterministic) — then the row factor f_i and, by
// the whole block, X'_i = bf16(f_i * x_i) for its rows (X'^T: one 16-byte store per column).
// 4 rows per block measured the same (0.74–0.76 ms per Llama-8B step with per-column stores); the
// 16-byte transpose below brought it to 0.63 ms.  The stash is not touched, except
// for rare rows where the per-row reference does not fit (a tile kept its own max, or f_i is
// outside [1e-30, 1e30]): those are rescaled in place to G_P tile by tile and get f_i = 1,
// X'_i = x_i.  xs may alias xrows (the fused RMSNorm's y buffer): each row is read then written by
// the same thread.
constexpr int CS_ROWS = 8, CS_LANES = 32;

__global__ void __launch_bounds__(256) combine_scale_kernel(
    const float2* __restrict__ partials, int tiles, int rows, const float* __restrict__ zt,
    const int32_t* __restrict__ t, int64_t V_l, int64_t ld_stash, int32_t ignore_index, int reduction, float scale,
    float grad_scale, const WsHeader* __restrict__ hdr, float* __restrict__ loss_rows,
    slf_rowstat* __restrict__ rowstat, uint16_t* __restrict__ stash, uint16_t* __restrict__ stash2, int split,
    const float* __restrict__ mref, float* __restrict__ fac, const uint16_t* xrows, uint16_t* xs, int64_t H,
    int64_t ld_xst, RmsStep rms, const slf_shardstat* __restrict__ st = nullptr, int g = 1, int64_t vocab_start = 0,
    int64_t V_global = 0) {
  // st (vocab shards): the row's lse comes from the g shards' statistics (shard order, as
  // combine_transform); this shard's tile partials still decide which of its tiles kept their max.
  // ld_xst > 0: X' is written transposed, X'^T [H][ld_xst] (the dW GEMM's B operand K-major)
  extern __shared__ float r_t[];  // [tiles]: per-tile factors of a fallback row
  griddep_launch_dependents();
  griddep_wait();  // PDL: everything below reads the previous kernel's outputs
  const int nblk = (rows + CS_ROWS - 1) / CS_ROWS;
  if ((int)blockIdx.x >= nblk) {  // the fused final RMSNorm's jobs riding in this launch (rmsnorm.cuh)
    rms_block(rms, (int64_t)blockIdx.x - nblk);
    return;
  }
  __shared__ float lm[CS_LANES][CS_ROWS], ls[CS_LANES][CS_ROWS];
  __shared__ int lfb[CS_LANES][CS_ROWS];
  __shared__ float sF[CS_ROWS], sLse[CS_ROWS], sCg[CS_ROWS];
  __shared__ int sFb[CS_ROWS];
  const int tid = threadIdx.x;
  const int rl = tid % CS_ROWS, lane = tid / CS_ROWS;
  const int i0 = blockIdx.x * CS_ROWS;
  {
    const int i = i0 + rl;
    float m = -INFINITY, sum = 0.f;
    int fb = 0;
    if (i < rows) {
      const float M = mref[i];
#pragma unroll 4
      for (int k = lane; k < tiles; k += CS_LANES) {
        const float2 p = partials[(size_t)k * rows + i];
        fb |= (p.x - M > STASH_REF_SLACK) ? 1 : 0;
        const float nm = fmaxf(m, p.x);
        sum = (m == -INFINITY ? 0.f : sum * ex2((m - nm) * LOG2E)) + p.y * ex2((p.x - nm) * LOG2E);
        m = nm;
      }
    }
    lm[lane][rl] = m;
    ls[lane][rl] = sum;
    lfb[lane][rl] = fb;
  }
  __syncthreads();
  if (tid < CS_ROWS && i0 + tid < rows) {  // one thread per row: lanes in order
    const int i = i0 + tid;
    float Mx = -INFINITY, S = 0.f;
    int fb = 0;
    for (int p = 0; p < CS_LANES; ++p) {
      Mx = fmaxf(Mx, lm[p][tid]);
      fb |= lfb[p][tid];
    }
    for (int p = 0; p < CS_LANES; ++p)
      if (lm[p][tid] != -INFINITY) S += ls[p][tid] * ex2((lm[p][tid] - Mx) * LOG2E);
    const int32_t tt = t[i];
    const int64_t Vg = st ? V_global : V_l;
    const bool valid = tt != ignore_index;
    const bool bad = valid && (tt < 0 || (int64_t)tt >= Vg);
    const int64_t loc = (int64_t)tt - vocab_start;
    const bool here = valid && !bad && loc >= 0 && loc < V_l;
    float z = here ? zt[i] : 0.f;
    if (st) {  // the global row statistics from the g shards, in shard order
      Mx = -INFINITY;
      S = 0.f;
      z = 0.f;
      for (int k = 0; k < g; ++k) Mx = fmaxf(Mx, st[(size_t)k * rows + i].m);
      for (int k = 0; k < g; ++k) {
        const slf_shardstat q = st[(size_t)k * rows + i];
        S += q.s * ex2((q.m - Mx) * LOG2E);
        z += q.zt;  // exactly one shard has the target (the others store 0)
      }
    }
    const float lse = Mx + logf(S);
    const float coef = (valid && !bad) ? coef_of(reduction, scale, hdr->n_valid) : 0.f;
    float l = valid ? (lse - z) : 0.f;
    if (bad) l = __int_as_float(0x7fc00000);
    loss_rows[i] = l;
    rowstat[i] = slf_rowstat{lse * LOG2E, coef, here ? (int32_t)loc : -1, valid ? 1 : 0};
    const float cg = coef * grad_scale;
    float f = 0.f;
    if (cg != 0.f) {
      f = cg * ex2((mref[i] - lse) * LOG2E);
      if (!(fabsf(f) >= 1e-30f && fabsf(f) <= 1e30f)) fb = 1;
    }
    sLse[tid] = lse;
    sCg[tid] = cg;
    sFb[tid] = fb;
    sF[tid] = fb ? 1.f : f;
    fac[i] = fb ? 1.f : f;
  }
  __syncthreads();
  for (int r = 0; r < CS_ROWS && i0 + r < rows; ++r) {  // rare: rescale a stash row in place to G_P
    if (!sFb[r]) continue;
    const int i = i0 + r;
    const float M = mref[i], lse = sLse[r], cg = sCg[r];
    for (int k = tid; k < tiles; k += 256) {
      const float mt = partials[(size_t)k * rows + i].x;
      float f;
      if (mt - M > STASH_REF_SLACK) f = cg * ex2((mt - lse) * LOG2E);  // the tile stored exp(z - m_t)
      else if (M - mt > 80.f) f = 0.f;                                 // its entries < e^-40 of the max
      else f = cg * ex2((M - mt) * LOG2E) * ex2((mt - lse) * LOG2E);    // it stored exp(z - M)
      r_t[k] = f;
    }
    __syncthreads();
    uint4* row = reinterpret_cast<uint4*>(i < split ? stash + (size_t)i * ld_stash
                                                    : stash2 + (size_t)(i - split) * ld_stash);
    const int64_t groups = (V_l + 7) / 8;
    for (int64_t q = tid; q < groups; q += 256) {
      const float f = r_t[(q * 8) / 256];
      uint4 x = row[q];
      x.x = pack_bf16x2(bf16lo_to_f32(x.x) * f, bf16hi_to_f32(x.x) * f);
      x.y = pack_bf16x2(bf16lo_to_f32(x.y) * f, bf16hi_to_f32(x.y) * f);
      x.z = pack_bf16x2(bf16lo_to_f32(x.z) * f, bf16hi_to_f32(x.z) * f);
      x.w = pack_bf16x2(bf16lo_to_f32(x.w) * f, bf16hi_to_f32(x.w) * f);
      row[q] = x;
    }
    __syncthreads();
  }
  // X'_i = bf16(f * x_i) for the block's rows (f = 1 for the rescaled rows: an exact copy); none
  // without a dW GEMM
  if (!xs) return;
  const int nr = min(CS_ROWS, rows - i0);
  if (ld_xst > 0 && CS_ROWS == 8 && nr == CS_ROWS) {
    // X'^T[h][i0 .. i0 + 8) for 8 consecutive columns h per thread: eight 16-byte row loads, a
    // register transpose, eight 16-byte column stores
    for (int64_t h0 = (int64_t)tid * 8; h0 < H; h0 += 256 * 8) {
      float v[CS_ROWS][8];
#pragma unroll
      for (int r = 0; r < CS_ROWS; ++r) {
        const uint4 q = *reinterpret_cast<const uint4*>(xrows + (size_t)(i0 + r) * H + h0);
        const float f = sF[r];
        v[r][0] = bf16lo_to_f32(q.x) * f; v[r][1] = bf16hi_to_f32(q.x) * f;
        v[r][2] = bf16lo_to_f32(q.y) * f; v[r][3] = bf16hi_to_f32(q.y) * f;
        v[r][4] = bf16lo_to_f32(q.z) * f; v[r][5] = bf16hi_to_f32(q.z) * f;
        v[r][6] = bf16lo_to_f32(q.w) * f; v[r][7] = bf16hi_to_f32(q.w) * f;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(xs + (size_t)(h0 + c) * ld_xst + i0) =
            make_uint4(pack_bf16x2(v[0][c], v[1][c]), pack_bf16x2(v[2][c], v[3][c]), pack_bf16x2(v[4][c], v[5][c]),
                       pack_bf16x2(v[6][c], v[7][c]));
    }
    return;
  }
  if (ld_xst > 0) {  // X'^T[h][i0 .. i0 + nr): CS_ROWS * 2 contiguous bytes per column h
    static_assert(CS_ROWS == 4 || CS_ROWS == 8, "one 8- or 16-byte store per column");
    for (int64_t h = tid; h < H; h += 256) {
      uint32_t w[CS_ROWS / 2];
#pragma unroll
      for (int r = 0; r < CS_ROWS; r += 2) {
        const float a = r < nr ? bf16_bits_to_f32(xrows[(size_t)(i0 + r) * H + h]) * sF[r] : 0.f;
        const float b = r + 1 < nr ? bf16_bits_to_f32(xrows[(size_t)(i0 + r + 1) * H + h]) * sF[r + 1] : 0.f;
        w[r / 2] = pack_bf16x2(a, b);
      }
      uint16_t* dst = xs + (size_t)h * ld_xst + i0;
      if (nr == CS_ROWS) {
        if constexpr (CS_ROWS == 8)
          *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[CS_ROWS / 2 - 2], w[CS_ROWS / 2 - 1]);
        else
          *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
      } else {
        for (int r = 0; r < nr; ++r) dst[r] = (uint16_t)(w[r / 2] >> ((r & 1) * 16));
      }
    }
    return;
  }
  const int64_t per_row = H / 8;
  for (int64_t q = tid; q < (int64_t)nr * per_row; q += 256) {
    const int r = (int)(q / per_row);
    const int64_t c = q - (int64_t)r * per_row;
    const float f = sF[r];
    const uint4 x = reinterpret_cast<const uint4*>(xrows + (size_t)(i0 + r) * H)[c];
    reinterpret_cast<uint4*>(xs + (size_t)(i0 + r) * H)[c] =
        make_uint4(pack_bf16x2(bf16lo_to_f32(x.x) * f, bf16hi_to_f32(x.x) * f),
                   pack_bf16x2(bf16lo_to_f32(x.y) * f, bf16hi_to_f32(x.y) * f),
                   pack_bf16x2(bf16lo_to_f32(x.z) * f, bf16hi_to_f32(x.z) * f),
                   pack_bf16x2(bf16lo_to_f32(x.w) * f, bf16hi_to_f32(x.w) * f));
  }
}

// ---- target CSR ------------------------------------------------------------------------------
__device__ __forceinline__ bool in_shard(int32_t tt, int32_t ignore_index, int64_t vocab_start, int64_t V_l) {
  const int64_t loc = (int64_t)tt - vocab_start;
  return tt != ignore_index && loc >= 0 && loc < V_l;
}

// X_chunk [rows][H] -> XT [H][ldxt] (bf16), so the dW GEMM's B operand (X_chunk, K = rows) can be
// K-major: with both dW operands MN-major the MMA issued ~9 % slower than with one.
// 64 x 64 tiles through shared memory, 16-byte loads and stores.  Launched with programmatic
// dependent launch after the previous group launch (whose extended stash it may overwrite).
__global__ void __launch_bounds__(256) transpose_x_kernel(const uint16_t* __restrict__ X, int64_t H, int rows,
                                                          uint16_t* __restrict__ XT, int64_t ldxt) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ uint16_t tile[64][72];
  const int i0 = blockIdx.x * 64, h0 = blockIdx.y * 64;
  for (int v = threadIdx.x; v < 512; v += 256) {
    const int r = v >> 3, c = (v & 7) * 8;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (i0 + r < rows && h0 + c < H) val = *reinterpret_cast<const uint4*>(X + (size_t)(i0 + r) * H + h0 + c);
    const uint16_t* e = reinterpret_cast<const uint16_t*>(&val);
#pragma unroll
    for (int k = 0; k < 8; ++k) tile[r][c + k] = e[k];
  }
  __syncthreads();
  for (int v = threadIdx.x; v < 512; v += 256) {
    const int hr = v >> 3, ic = (v & 7) * 8;
    if (h0 + hr >= H || i0 + ic >= rows) continue;
    uint16_t e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = tile[ic + k][hr];
    *reinterpret_cast<uint4*>(XT + (size_t)(h0 + hr) * ldxt + i0 + ic) = *reinterpret_cast<const uint4*>(e);
  }
}

__global__ void csr_zero_kernel(int32_t* __restrict__ cnt, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = 0;
}

__global__ void csr_count_kernel(const int32_t* __restrict__ t, int64_t N, int32_t ignore_index, int64_t vocab_start,
                                 int64_t V_l, int32_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N && in_shard(t[i], ignore_index, vocab_start, V_l)) atomicAdd(&cnt[t[i] - vocab_start], 1);
}

// Single block: off = exclusive_scan(cnt) over V_l entries (off[V_l] = total); hit list of rows with
// cnt > 0 in increasing row order; n_hits stored in off[V_l + 1].  Each pass covers 8192
// consecutive entries: eight per thread (coalesced loads, all in flight at once), a serial scan of
// the thread's eight, warp-shuffle scans of the thread totals and a running carry (integer, exact).
constexpr int CSR_SCAN_SPAN = 8192;

// Multi-block form, first kernel: per span of 8192 entries, (sum of counts, number of nonzero).
__global__ void __launch_bounds__(1024) csr_blocksum_kernel(const int32_t* __restrict__ cnt, int64_t V_l,
                                                           int2* __restrict__ bsum) {
  __shared__ int32_t ws[32], wh[32];
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * CSR_SCAN_SPAN;
  int32_t s = 0, h = 0;
#pragma unroll
  for (int k = 0; k < CSR_SCAN_SPAN / 1024; ++k) {
    const int64_t v = base + k * 1024 + tid;
    const int32_t c = v < V_l ? cnt[v] : 0;
    s += c;
    h += c > 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    h += __shfl_xor_sync(0xffffffffu, h, o);
  }
  if ((tid & 31) == 0) {
    ws[tid >> 5] = s;
    wh[tid >> 5] = h;
  }
  __syncthreads();
  if (tid == 0) {
    int32_t S = 0, Hh = 0;
    for (int w = 0; w < 32; ++w) {
      S += ws[w];
      Hh += wh[w];
    }
    bsum[blockIdx.x] = make_int2(S, Hh);
  }
}

// With bsum == nullptr: one block scans all spans in turn (a running carry).  With bsum (from
// csr_blocksum_kernel): block b scans span b only, starting from the sum of the earlier spans'
// totals; the last block writes the totals.  Integer, exact, the same result either way.
__global__ void __launch_bounds__(1024) csr_scan_kernel(const int32_t* __restrict__ cnt, int64_t V_l,
                                                       int32_t* __restrict__ off, int32_t* __restrict__ hits,
                                                       const int2* __restrict__ bsum = nullptr) {
  constexpr int PER = 8, SPAN = 1024 * PER;
  static_assert(SPAN == CSR_SCAN_SPAN, "span");
  __shared__ int32_t stage[SPAN];
  __shared__ int32_t wsum[32], whit[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t carry_s = 0, carry_h = 0;  // identical in every thread
  int64_t b0 = 0, b1 = V_l;
  if (bsum) {
    b0 = (int64_t)blockIdx.x * SPAN;
    b1 = min(V_l, b0 + SPAN);
    for (int b = 0; b < (int)blockIdx.x; ++b) {  // fixed order, every thread (<= V/8192 entries)
      const int2 q = bsum[b];
      carry_s += q.x;
      carry_h += q.y;
    }
  }
  for (int64_t base = b0; base < b1; base += SPAN) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {  // coalesced: entry base + k*1024 + tid
      const int64_t v = base + k * 1024 + tid;
      stage[k * 1024 + tid] = v < V_l ? cnt[v] : 0;
    }
    __syncthreads();
    int32_t c[PER], s = 0, h = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {  // this thread's eight consecutive entries
      c[k] = stage[tid * PER + k];
      s += c[k];
      h += c[k] > 0;
    }
    int32_t si = s, hi = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t a = __shfl_up_sync(0xffffffffu, si, o), b2 = __shfl_up_sync(0xffffffffu, hi, o);
      if (lane >= o) {
        si += a;
        hi += b2;
      }
    }
    if (lane == 31) {
      wsum[warp] = si;
      whit[warp] = hi;
    }
    __syncthreads();
    if (warp == 0) {
      int32_t ws = wsum[lane], wh = whit[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t a = __shfl_up_sync(0xffffffffu, ws, o), b2 = __shfl_up_sync(0xffffffffu, wh, o);
        if (lane >= o) {
          ws += a;
          wh += b2;
        }
      }
      wsum[lane] = ws;  // inclusive over warps
      whit[lane] = wh;
    }
    __syncthreads();
    int32_t ps = carry_s + (warp ? wsum[warp - 1] : 0) + si - s;
    int32_t ph = carry_h + (warp ? whit[warp - 1] : 0) + hi - h;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int64_t v = base + (int64_t)tid * PER + k;
      if (v < V_l) {
        off[v] = ps;
        if (c[k] > 0) hits[ph++] = (int32_t)v;
      }
      ps += c[k];
    }
    carry_s += wsum[31];
    carry_h += whit[31];
    __syncthreads();  // stage / wsum / whit are rewritten by the next pass
  }
  if (tid == 0 && (bsum == nullptr || blockIdx.x == gridDim.x - 1)) {
    off[V_l] = carry_s;
    off[V_l + 1] = carry_h;
  }
}

// rank_i = #{j < i : t_j == t_i, both in shard}; idx[off[t_i] + rank_i] = i.  Brute force over
// earlier tokens through shared-memory tiles (only for targets that occur more than once); four
// lanes per token each count a quarter of every tile, summed with shuffles (integer, exact).
constexpr int CSR_TOK_PER_BLOCK = 64;
__global__ void __launch_bounds__(256) csr_scatter_kernel(const int32_t* __restrict__ t, int64_t N,
                                                         int32_t ignore_index, int64_t vocab_start, int64_t V_l,
                                                         const int32_t* __restrict__ cnt,
                                                         const int32_t* __restrict__ off, int32_t* __restrict__ idx) {
  __shared__ int32_t tile[2048];
  const int part = threadIdx.x & 3;
  const int64_t i = (int64_t)blockIdx.x * CSR_TOK_PER_BLOCK + (threadIdx.x >> 2);
  int32_t key = -1;
  bool need = false;
  if (i < N && in_shard(t[i], ignore_index, vocab_start, V_l)) {
    key = t[i];
    need = cnt[key - vocab_start] > 1;
  }
  const int any_need = __syncthreads_or(need);
  int32_t rank = 0;
  if (any_need) {
    const int64_t end = (int64_t)blockIdx.x * CSR_TOK_PER_BLOCK + CSR_TOK_PER_BLOCK;  // tokens before the last
    for (int64_t j0 = 0; j0 < end && j0 < N; j0 += 2048) {
      for (int k = threadIdx.x; k < 2048; k += blockDim.x) tile[k] = (j0 + k < N) ? t[j0 + k] : ignore_index;
      __syncthreads();
      if (need) {
        const int64_t rem = i - j0;
        const int lim = rem < 2048 ? (int)rem : 2048;
        for (int k = part; k < lim; k += 4) rank += (tile[k] == key);
      }
      __syncthreads();
    }
  }
  rank += __shfl_xor_sync(0xffffffffu, rank, 1);
  rank += __shfl_xor_sync(0xffffffffu, rank, 2);
  if (key >= 0 && part == 0) idx[off[key - vocab_start] + rank] = (int32_t)i;  // valid and in shard
}

// ---- stable rank by block sort + binary search (replaces the brute-force rank above when the
// workspace has scratch for N packed keys).  rank_i = #{j < i : t_j = t_i} is split
// as (earlier token blocks) + (earlier tokens of i's own block).  Kernel 1 sorts each block of
// CSR_SORT_T tokens by the packed key (t_i - vocab_start) << 12 | (i mod T) in shared memory
// (bitonic; the packed keys are unique, so the order is the stable order by target); tokens that
// are ignored or outside the shard sort last as 0xffffffff.  Kernel 2 counts, for a token with a
// repeated target, the entries of its key in every earlier block and its own block's entries
// before it with binary searches on the sorted blocks.  Integer and exact; no atomics decide
// positions.  Needs V_l < 2^20.
constexpr int CSR_SORT_T = 4096, CSR_SORT_SHIFT = 12;

__global__ void __launch_bounds__(1024) csr_block_sort_kernel(const int32_t* __restrict__ t, int64_t N,
                                                             int32_t ignore_index, int64_t vocab_start, int64_t V_l,
                                                             uint32_t* __restrict__ sorted) {
  __shared__ uint32_t k[CSR_SORT_T];
  const int64_t b0 = (int64_t)blockIdx.x * CSR_SORT_T;
#pragma unroll
  for (int e = 0; e < CSR_SORT_T / 1024; ++e) {
    const int li = e * 1024 + threadIdx.x;
    const int64_t i = b0 + li;
    uint32_t v = 0xffffffffu;
    if (i < N) {
      const int32_t tt = t[i];
      if (in_shard(tt, ignore_index, vocab_start, V_l))
        v = ((uint32_t)(tt - vocab_start) << CSR_SORT_SHIFT) | (uint32_t)li;
    }
    k[li] = v;
  }
  __syncthreads();
  for (int size = 2; size <= CSR_SORT_T; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int e = 0; e < CSR_SORT_T / 2048; ++e) {
        const int j = e * 1024 + threadIdx.x;               // compare-exchange pair j of T/2
        const int lo = 2 * j - (j & (stride - 1));          // first index of the pair
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint32_t a = k[lo], b = k[hi];
        if ((a > b) == up) {
          k[lo] = b;
          k[hi] = a;
        }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int e = 0; e < CSR_SORT_T / 1024; ++e) sorted[b0 + e * 1024 + threadIdx.x] = k[e * 1024 + threadIdx.x];
}

__device__ __forceinline__ int lower_bound_u32(const uint32_t* __restrict__ a, int n, uint32_t x) {
  int lo = 0;
  while (n > 0) {
    const int h = n >> 1;
    if (__ldg(a + lo + h) < x) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo;
}

__global__ void __launch_bounds__(256) csr_rank_scatter_kernel(const int32_t* __restrict__ t, int64_t N,
                                                              int32_t ignore_index, int64_t vocab_start, int64_t V_l,
                                                              const int32_t* __restrict__ cnt,
                                                              const int32_t* __restrict__ off,
                                                              const uint32_t* __restrict__ sorted,
                                                              int32_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int32_t tt = t[i];
  if (!in_shard(tt, ignore_index, vocab_start, V_l)) return;
  const uint32_t key = (uint32_t)(tt - vocab_start);
  int32_t rank = 0;
  if (cnt[key] > 1) {
    const uint32_t k0 = key << CSR_SORT_SHIFT, k1 = (key + 1) << CSR_SORT_SHIFT;
    const int64_t b = i / CSR_SORT_T;
    for (int64_t bb = 0; bb < b; ++bb) {  // every earlier block: its entries with this key
      const uint32_t* blk = sorted + bb * CSR_SORT_T;
      rank += lower_bound_u32(blk, CSR_SORT_T, k1) - lower_bound_u32(blk, CSR_SORT_T, k0);
    }
    const uint32_t* own = sorted + b * CSR_SORT_T;  // own block: entries of this key before token i
    rank += lower_bound_u32(own, CSR_SORT_T, k0 | (uint32_t)(i - b * CSR_SORT_T)) - lower_bound_u32(own, CSR_SORT_T, k0);
  }
  idx[off[key] + rank] = (int32_t)i;
}

// ---- one-hot dW correction, segmented: dW[v] -= coef * sum_{t_i = v} x_i.
// The CSR positions [0, n) (sorted by target, then token) are cut into segments of S positions;
// pass 1 (one block per segment and 1024-column slab) walks its positions in order, summing x in
// fp32 per target row: a row that starts and ends inside the segment is applied to dW at once;
// the part of a row that continues from the previous segment goes to partial slot 0 of the
// segment, the part of a row that starts here and continues to slot 1.  Pass 2: the segment where
// such a row starts sums its slot 1 and the following segments' slot 0 in segment order and
// applies it.  Each row's sum is therefore fp32 in token order within segments, the segment sums
// added left to right: fixed order, deterministic, and a hot row (thousands of hits under Zipf
// targets) is spread over many blocks instead of one block's serial loop.
__device__ __forceinline__ void onehot_apply(uint16_t* __restrict__ dW, int64_t H, int32_t v, int64_t col, float c,
                                             const float* acc) {
  uint4* d = reinterpret_cast<uint4*>(dW + (size_t)v * H + col);
  const uint4 o = *d;
  *d = make_uint4(pack_bf16x2(bf16lo_to_f32(o.x) - c * acc[0], bf16hi_to_f32(o.x) - c * acc[1]),
                  pack_bf16x2(bf16lo_to_f32(o.y) - c * acc[2], bf16hi_to_f32(o.y) - c * acc[3]),
                  pack_bf16x2(bf16lo_to_f32(o.z) - c * acc[4], bf16hi_to_f32(o.z) - c * acc[5]),
                  pack_bf16x2(bf16lo_to_f32(o.w) - c * acc[6], bf16hi_to_f32(o.w) - c * acc[7]));
}

// The CSR row holding position p: the largest r with off[r] <= p (its off[r + 1] > p, so r has hits).
__device__ __forceinline__ int32_t csr_row_of(const int32_t* __restrict__ off, int64_t V_l, int64_t p) {
  int64_t lo = 0, n = V_l;  // search off[0 .. V_l): first index with off > p, minus one
  while (n > 0) {
    const int64_t h = n >> 1;
    if (off[lo + h] <= p) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return (int32_t)(lo - 1);
}

// The hit-row index holding position p: the largest h with off[hits[h]] <= p (hits: the rows with
// at least one token, increasing; n_hits of them).
__device__ __forceinline__ int64_t csr_hit_of(const int32_t* __restrict__ off, const int32_t* __restrict__ hits,
                                              int64_t n_hits, int64_t p) {
  int64_t lo = 0, n = n_hits;
  while (n > 0) {
    const int64_t h = n >> 1;
    if (off[hits[lo + h]] <= p) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo - 1;
}

__global__ void __launch_bounds__(128) onehot_seg_kernel(const uint16_t* __restrict__ X, int64_t H,
                                                        const int32_t* __restrict__ off,
                                                        const int32_t* __restrict__ hits,
                                                        const int32_t* __restrict__ idx, int64_t V_l, int S,
                                                        int reduction, float scale, float grad_scale,
                                                        const WsHeader* __restrict__ hdr, float* __restrict__ part,
                                                        uint16_t* __restrict__ dW, const float* __restrict__ rstd,
                                                        const uint16_t* __restrict__ gam) {
  // rstd / gam (fused final RMSNorm, else null): the GEMMs' rows are y = bf16(x * rstd * g), so the
  // one-hot term sums exactly those bf16 values, recomputed here with the forward's fp32 ops.
  const int64_t n = off[V_l];
  const int64_t p0 = (int64_t)blockIdx.x * S;
  if (p0 >= n) return;
  const int64_t p1 = min(p0 + (int64_t)S, n);
  const int64_t col = ((int64_t)blockIdx.y * 128 + threadIdx.x) * 8;
  if (col >= H) return;
  const float c = coef_of(reduction, scale, hdr->n_valid) * grad_scale;
  float gw[8];
  if (rstd) {
    const uint4 q = *reinterpret_cast<const uint4*>(gam + col);
    gw[0] = bf16lo_to_f32(q.x); gw[1] = bf16hi_to_f32(q.x); gw[2] = bf16lo_to_f32(q.y); gw[3] = bf16hi_to_f32(q.y);
    gw[4] = bf16lo_to_f32(q.z); gw[5] = bf16hi_to_f32(q.z); gw[6] = bf16lo_to_f32(q.w); gw[7] = bf16hi_to_f32(q.w);
  }
  // rows in position order are consecutive entries of the hit list: one search per segment, then
  // the next row is hits[h + 1] (round 2's first version searched the offsets at every row change)
  int64_t h = csr_hit_of(off, hits, off[V_l + 1], p0);
  int32_t row = hits[h];
  int64_t row_beg = off[row], row_end = off[row + 1];
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t p = p0; p < p1; ++p) {
    const int32_t tok = idx[p];
    uint4 x = *reinterpret_cast<const uint4*>(X + (size_t)tok * H + col);
    if (rstd) {
      const float r = rstd[tok];
      x = make_uint4(pack_bf16x2(bf16lo_to_f32(x.x) * r * gw[0], bf16hi_to_f32(x.x) * r * gw[1]),
                     pack_bf16x2(bf16lo_to_f32(x.y) * r * gw[2], bf16hi_to_f32(x.y) * r * gw[3]),
                     pack_bf16x2(bf16lo_to_f32(x.z) * r * gw[4], bf16hi_to_f32(x.z) * r * gw[5]),
                     pack_bf16x2(bf16lo_to_f32(x.w) * r * gw[6], bf16hi_to_f32(x.w) * r * gw[7]));
    }
    acc[0] += bf16lo_to_f32(x.x); acc[1] += bf16hi_to_f32(x.x);
    acc[2] += bf16lo_to_f32(x.y); acc[3] += bf16hi_to_f32(x.y);
    acc[4] += bf16lo_to_f32(x.z); acc[5] += bf16hi_to_f32(x.z);
    acc[6] += bf16lo_to_f32(x.w); acc[7] += bf16hi_to_f32(x.w);
    if (p + 1 == row_end || p + 1 == p1) {
      if (row_beg >= p0 && row_end <= p1) {
        onehot_apply(dW, H, row, col, c, acc);
      } else {
        float* dst = part + ((size_t)blockIdx.x * 2 + (row_beg < p0 ? 0 : 1)) * H + col;
        *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.f;
      if (p + 1 < p1) {
        row = hits[++h];
        row_beg = off[row];
        row_end = off[row + 1];
      }
    }
  }
}

__global__ void __launch_bounds__(128) onehot_join_kernel(int64_t H, const int32_t* __restrict__ off, int64_t V_l, int S,
                                                         int reduction, float scale, float grad_scale,
                                                         const WsHeader* __restrict__ hdr,
                                                         const float* __restrict__ part, uint16_t* __restrict__ dW) {
  const int64_t n = off[V_l];
  const int64_t p0 = (int64_t)blockIdx.x * S;
  if (p0 >= n) return;
  const int64_t p1 = min(p0 + (int64_t)S, n);
  const int32_t row = csr_row_of(off, V_l, p1 - 1);  // the segment's last row
  const int64_t row_beg = off[row], row_end = off[row + 1];
  if (row_beg < p0 || row_end <= p1) return;  // it does not start here, or ends inside: not ours
  const int64_t col = ((int64_t)blockIdx.y * 128 + threadIdx.x) * 8;
  if (col >= H) return;
  float acc[8];
  {
    const float* src = part + ((size_t)blockIdx.x * 2 + 1) * H + col;
    const float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + 4);
    acc[0] = a.x; acc[1] = a.y; acc[2] = a.z; acc[3] = a.w; acc[4] = b.x; acc[5] = b.y; acc[6] = b.z; acc[7] = b.w;
  }
  const int64_t q_last = (row_end - 1) / S;
  for (int64_t q = blockIdx.x + 1; q <= q_last; ++q) {  // following segments' continuation parts, in order
    const float* src = part + ((size_t)q * 2) * H + col;
    const float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + 4);
    acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
    acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
  }
  onehot_apply(dW, H, row, col, coef_of(reduction, scale, hdr->n_valid) * grad_scale, acc);
}

// dW[v] = bf16( f32(dW[v]) - coef * sum_{i in CSR[v]} x_i ), sums in fp32 in token order.
// grid.x over hit rows (bounded by min(N, V_l); n_hits in off[V_l + 1]), grid.y over 1024-column slabs.
__global__ void __launch_bounds__(128) onehot_kernel(const uint16_t* __restrict__ X, int64_t H,
                                                    const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                                                    const int32_t* __restrict__ hits, int64_t V_l, int reduction,
                                                    float scale, float grad_scale, const WsHeader* __restrict__ hdr,
                                                    uint16_t* __restrict__ dW) {
  const int64_t k = blockIdx.x;
  if (k >= off[V_l + 1]) return;
  const int32_t v = hits[k];
  const int64_t col = ((int64_t)blockIdx.y * 128 + threadIdx.x) * 8;
  if (col >= H) return;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int32_t p = off[v]; p < off[v + 1]; ++p) {
    const uint4 x = *reinterpret_cast<const uint4*>(X + (size_t)idx[p] * H + col);
    acc[0] += bf16lo_to_f32(x.x); acc[1] += bf16hi_to_f32(x.x);
    acc[2] += bf16lo_to_f32(x.y); acc[3] += bf16hi_to_f32(x.y);
    acc[4] += bf16lo_to_f32(x.z); acc[5] += bf16hi_to_f32(x.z);
    acc[6] += bf16lo_to_f32(x.w); acc[7] += bf16hi_to_f32(x.w);
  }
  const float c = coef_of(reduction, scale, hdr->n_valid) * grad_scale;
  uint4* d = reinterpret_cast<uint4*>(dW + (size_t)v * H + col);
  const uint4 o = *d;
  *d = make_uint4(pack_bf16x2(bf16lo_to_f32(o.x) - c * acc[0], bf16hi_to_f32(o.x) - c * acc[1]),
                  pack_bf16x2(bf16lo_to_f32(o.y) - c * acc[2], bf16hi_to_f32(o.y) - c * acc[3]),
                  pack_bf16x2(bf16lo_to_f32(o.z) - c * acc[4], bf16hi_to_f32(o.z) - c * acc[5]),
                  pack_bf16x2(bf16lo_to_f32(o.w) - c * acc[6], bf16hi_to_f32(o.w) - c * acc[7]));
}

// Single block: deterministic sum (fixed strided subsets + fixed tree, fp64) of the row losses.
__global__ void __launch_bounds__(1024) loss_reduce_kernel(const float* __restrict__ loss_rows, int64_t N,
                                                          int reduction, const WsHeader* __restrict__ hdr,
                                                          float* __restrict__ loss_out) {
  __shared__ double sh[1024];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += 1024) a += (double)loss_rows[i];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double tot = sh[0];
    const unsigned long long nv = hdr->n_valid;
    if (reduction == SLF_MEAN) tot = nv ? tot / (double)nv : 0.0;
    loss_out[0] = hdr->bad > 0 ? __int_as_float(0x7fc00000) : (float)tot;
  }
}

}  // namespace slf
