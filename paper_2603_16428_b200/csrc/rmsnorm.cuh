// rmsnorm.cuh — the final RMSNorm that feeds the LM head (the paper ships a
// Triton RMSNorm kernel beside the fused LCE).  HBM-bound, one block per row.
//   forward : y = bf16(x * rstd * g),  rstd = 1 / sqrt(mean(x^2) + eps)      (rstd kept in fp32)
//   backward: dx = rstd * (g*dy - xhat * mean(xhat * g*dy)),  xhat = x * rstd
//             dg = sum_rows dy * xhat   (per-block fp32 partials, then a fixed-order column sum)
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace slf {

constexpr int RMS_THREADS = 256;

__device__ __forceinline__ float block_sum_256(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < RMS_THREADS / 32; ++i) t += red[i];  // fixed order
  __syncthreads();
  return t;
}

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }

__device__ __forceinline__ void unpack8(const uint4 q, float (&f)[8]) {
  f[0] = bf16lo_to_f32(q.x); f[1] = bf16hi_to_f32(q.x);
  f[2] = bf16lo_to_f32(q.y); f[3] = bf16hi_to_f32(q.y);
  f[4] = bf16lo_to_f32(q.z); f[5] = bf16hi_to_f32(q.z);
  f[6] = bf16lo_to_f32(q.w); f[7] = bf16hi_to_f32(q.w);
}

// grid = N rows.  H % 8 == 0.
__global__ void __launch_bounds__(RMS_THREADS) rmsnorm_fwd_kernel(const uint16_t* __restrict__ x,
                                                                 const uint16_t* __restrict__ g, int64_t H, float eps,
                                                                 uint16_t* __restrict__ y, float* __restrict__ rstd) {
  __shared__ float red[RMS_THREADS / 32];
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
  const int64_t groups = H / 8;
  float ss = 0.f;
  for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
    float f[8];
    unpack8(xr[q], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
  }
  const float r = rsqrtf(block_sum_256(ss, red) / (float)H + eps);
  if (threadIdx.x == 0) rstd[row] = r;
  uint4* yr = reinterpret_cast<uint4*>(y + row * H);
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
    float f[8], w[8];
    unpack8(xr[q], f);
    unpack8(gr[q], w);
    yr[q] = make_uint4(pack_bf16x2(f[0] * r * w[0], f[1] * r * w[1]), pack_bf16x2(f[2] * r * w[2], f[3] * r * w[3]),
                       pack_bf16x2(f[4] * r * w[4], f[5] * r * w[5]), pack_bf16x2(f[6] * r * w[6], f[7] * r * w[7]));
  }
}

// grid = ceil(N / rows_per_block).  dy (bf16) and dx (bf16) may alias (in place, row-owned).
// dg_part [gridDim.x][H] fp32.
__global__ void __launch_bounds__(RMS_THREADS) rmsnorm_bwd_kernel(const uint16_t* __restrict__ x,
                                                                 const uint16_t* __restrict__ g,
                                                                 const float* __restrict__ rstd, const uint16_t* dy,
                                                                 int64_t N, int64_t H, int rows_per_block,
                                                                 uint16_t* dx, float* __restrict__ dg_part) {
  __shared__ float red[RMS_THREADS / 32];
  extern __shared__ float dg_acc[];  // [H] per-block partial of dg
  const int64_t groups = H / 8;
  for (int64_t j = threadIdx.x; j < H; j += RMS_THREADS) dg_acc[j] = 0.f;
  __syncthreads();
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  for (int64_t row = r0; row < r0 + rows_per_block && row < N; ++row) {
    const float r = rstd[row];
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
    const uint4* dr = reinterpret_cast<const uint4*>(dy + row * H);
    float dot = 0.f;
    for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
      float f[8], w[8], d[8];
      unpack8(xr[q], f);
      unpack8(gr[q], w);
      unpack8(dr[q], d);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = f[e] * r;
        dot = fmaf(xh, w[e] * d[e], dot);
        dg_acc[q * 8 + e] += d[e] * xh;  // thread-owned columns: no race
      }
    }
    const float c = block_sum_256(dot, red) / (float)H;
    uint4* xo = reinterpret_cast<uint4*>(dx + row * H);
    for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
      float f[8], w[8], d[8], o[8];
      unpack8(xr[q], f);
      unpack8(gr[q], w);
      unpack8(dr[q], d);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = r * (w[e] * d[e] - f[e] * r * c);
      xo[q] = make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]), pack_bf16x2(o[4], o[5]),
                         pack_bf16x2(o[6], o[7]));
    }
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < H; j += RMS_THREADS) dg_part[(size_t)blockIdx.x * H + j] = dg_acc[j];
}

// dg[j] = sum_b dg_part[b][j] in block order (deterministic); fp32 out.
__global__ void __launch_bounds__(256) rmsnorm_dg_reduce_kernel(const float* __restrict__ dg_part, int nblk,
                                                               int64_t H, float* __restrict__ dg) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  float s = 0.f;
  for (int b = 0; b < nblk; ++b) s += dg_part[(size_t)b * H + j];
  dg[j] = s;
}

// ---- final RMSNorm fused into the schedule-S chunk loop (slf_rmsnorm_lce_fwd_bwd) ----
// The RMSNorm work of the chunk loop rides in the blocks of launches the loop makes anyway (chunk
// k's combine_transform, which waits for chunk k's stash GEMM and hence for chunk k-1's grouped
// GEMMs), so the fusion adds no kernel boundary per chunk.  Jobs, by block range after the host
// launch's own blocks:
//   dx   chunk k-2: dx = rstd * (g*dy - xhat * mean(xhat*g*dy)) in place over dy (the group's bf16
//        dX output in the caller's dx rows; its dg partial was taken one launch earlier)   1 row / block
//   dgp  chunk k-1: part[rowgroup][col] = sum over the group's RMS_RG rows of dy * xhat, in row
//        order                                                       (row group x 256 columns) / block
//   fwd  chunk k+1: y = bf16(x * rstd * g) into its chunk buffer (double-buffered by parity), rstd  1 row / block
//   red  chunk k-2: dg (+)= sum over its row groups of part, in row-group order    256 columns / block
// Every job reads only what an earlier, completed launch wrote; y never exists for all N rows.
constexpr int RMS_RG = 32;  // rows per dg partial

struct RmsStep {
  const uint16_t* x;
  const uint16_t* g;
  int64_t H;
  float eps;
  float* rstd;    // [N]
  uint16_t* dx;   // [N][H]: dy in, dx out (row-owned, in place)
  int64_t x_r0, x_rows;     // dx job rows
  int64_t p_r0, p_rows;     // dg-partial job rows
  float* part_w;            // [ceil(p_rows / RMS_RG)][H]
  int64_t f_r0, f_rows;     // fwd job rows
  uint16_t* ybuf;           // [f_rows][H]
  int red_ngroups, red_first;  // red job: row groups to sum (0: none)
  const float* part_r;
  float* dg;
  // fwd job, per-row stash reference (s_kernels.cuh mref_kernel; null: not needed): mref[row] =
  // y_row . W[t_row] + shift, or +inf for ignored / out-of-range targets
  const uint16_t* W;
  const int32_t* t;
  int32_t ignore_index;
  int64_t V;
  float shift;
  float* mref;
};

__host__ __device__ inline int rms_nslab(int64_t H) { return (int)((H + 255) / 256); }
__host__ __device__ inline int64_t rms_blocks_of(const RmsStep& a) {
  const int slabs = rms_nslab(a.H);
  return a.x_rows + ((a.p_rows + RMS_RG - 1) / RMS_RG) * slabs + a.f_rows + (a.red_ngroups ? slabs : 0);
}

__device__ __forceinline__ void rms_block(const RmsStep& a, int64_t b) {
  __shared__ float red[RMS_THREADS / 32];
  const int64_t groups = a.H / 8;
  const uint4* gr = reinterpret_cast<const uint4*>(a.g);
  const int slabs = rms_nslab(a.H);
  if (b < a.x_rows) {  // dx of one row, in place
    const int64_t row = a.x_r0 + b;
    const float r = a.rstd[row];
    const uint4* xr = reinterpret_cast<const uint4*>(a.x + row * a.H);
    uint4* dr = reinterpret_cast<uint4*>(a.dx + row * a.H);
    float dot = 0.f;
    for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
      float f[8], w[8], d[8];
      unpack8(xr[q], f);
      unpack8(gr[q], w);
      unpack8(dr[q], d);
#pragma unroll
      for (int e = 0; e < 8; ++e) dot = fmaf(f[e] * r, w[e] * d[e], dot);
    }
    const float c = block_sum_256(dot, red) / (float)a.H;
    for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
      float f[8], w[8], d[8], o[8];
      unpack8(xr[q], f);
      unpack8(gr[q], w);
      unpack8(dr[q], d);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = r * (w[e] * d[e] - f[e] * r * c);
      dr[q] = make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]), pack_bf16x2(o[4], o[5]),
                         pack_bf16x2(o[6], o[7]));
    }
    return;
  }
  b -= a.x_rows;
  const int64_t npb = ((a.p_rows + RMS_RG - 1) / RMS_RG) * slabs;
  if (b < npb) {  // dg partial: one row group x 256 columns, thread = column, rows in order
    const int64_t grp = b / slabs;
    const int64_t col = (b % slabs) * 256 + threadIdx.x;
    if (col >= a.H) return;
    const int64_t r0 = a.p_r0 + grp * RMS_RG, r1 = min(r0 + RMS_RG, a.p_r0 + a.p_rows);
    float acc = 0.f;
#pragma unroll 8
    for (int64_t row = r0; row < r1; ++row) {
      const float xv = bf16_bits_to_f32(a.x[row * a.H + col]) * a.rstd[row];
      acc += bf16_bits_to_f32(a.dx[row * a.H + col]) * xv;
    }
    a.part_w[grp * a.H + col] = acc;
    return;
  }
  b -= npb;
  if (b < a.f_rows) {  // forward of one row
    const int64_t row = a.f_r0 + b;
    const uint4* xr = reinterpret_cast<const uint4*>(a.x + row * a.H);
    float ss = 0.f;
    for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
      float f[8];
      unpack8(xr[q], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
    }
    const float r = rsqrtf(block_sum_256(ss, red) / (float)a.H + a.eps);
    if (threadIdx.x == 0) a.rstd[row] = r;
    uint4* yr = reinterpret_cast<uint4*>(a.ybuf + b * a.H);
    int64_t loc = -1;
    if (a.mref) {
      const int32_t tt = a.t[row];
      loc = (tt == a.ignore_index || tt < 0 || (int64_t)tt >= a.V) ? -1 : (int64_t)tt;
    }
    const uint4* wr = reinterpret_cast<const uint4*>(a.W + (loc >= 0 ? loc : 0) * a.H);
    float dot = 0.f;
    for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
      float f[8], w[8];
      unpack8(xr[q], f);
      unpack8(gr[q], w);
      const uint4 y = make_uint4(pack_bf16x2(f[0] * r * w[0], f[1] * r * w[1]), pack_bf16x2(f[2] * r * w[2], f[3] * r * w[3]),
                                 pack_bf16x2(f[4] * r * w[4], f[5] * r * w[5]), pack_bf16x2(f[6] * r * w[6], f[7] * r * w[7]));
      yr[q] = y;
      if (loc >= 0) {
        float yv[8], wv[8];
        unpack8(y, yv);
        unpack8(wr[q], wv);
#pragma unroll
        for (int e = 0; e < 8; ++e) dot = fmaf(yv[e], wv[e], dot);
      }
    }
    if (a.mref) {
      const float d = block_sum_256(dot, red);  // block-uniform branch (loc is per row)
      if (threadIdx.x == 0) a.mref[row] = loc >= 0 ? d + a.shift : INFINITY;
    }
    return;
  }
  b -= a.f_rows;
  const int64_t col = b * 256 + threadIdx.x;  // dg reduction of one 256-column slab
  if (col >= a.H) return;
  float sum = 0.f;
  for (int k = 0; k < a.red_ngroups; ++k) sum += a.part_r[(size_t)k * a.H + col];
  a.dg[col] = a.red_first ? sum : a.dg[col] + sum;
}

// Standalone form (the loop's first forward and its tail), programmatic dependent launch.
__global__ void __launch_bounds__(RMS_THREADS) rms_step_kernel(RmsStep a) {
  griddep_launch_dependents();
  griddep_wait();
  rms_block(a, blockIdx.x);
}

// p[i] = bf16(p[i] * s), 8 elements per thread-iteration.
__global__ void __launch_bounds__(256) scale_bf16_kernel(uint4* __restrict__ p, int64_t groups, float s) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < groups; q += (int64_t)gridDim.x * blockDim.x) {
    float f[8];
    unpack8(p[q], f);
    p[q] = make_uint4(pack_bf16x2(f[0] * s, f[1] * s), pack_bf16x2(f[2] * s, f[3] * s), pack_bf16x2(f[4] * s, f[5] * s),
                      pack_bf16x2(f[6] * s, f[7] * s));
  }
}

// p[i] = bf16(p[i] * s[0]) with the factor on the device (an autograd grad_output, no host read);
// every block returns at once when it is exactly 1 (the common loss.backward()).
__global__ void __launch_bounds__(256) scale_bf16_dev_kernel(uint4* __restrict__ p, int64_t groups,
                                                            const float* __restrict__ s_dev) {
  const float s = *s_dev;
  if (s == 1.0f) return;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < groups; q += (int64_t)gridDim.x * blockDim.x) {
    float f[8];
    unpack8(p[q], f);
    p[q] = make_uint4(pack_bf16x2(f[0] * s, f[1] * s), pack_bf16x2(f[2] * s, f[3] * s), pack_bf16x2(f[4] * s, f[5] * s),
                      pack_bf16x2(f[6] * s, f[7] * s));
  }
}

// RowStat out[i] = in[i] with coef *= grad[per_row ? i : 0]: the upstream gradient of the loss
// (scalar for SUM/MEAN, per row for NONE) folded into the backward's per-row coefficient, on the
// device.  in / out: 16-byte records {lse2, coef, tloc, valid}.
__global__ void __launch_bounds__(256) rowstat_scale_kernel(const float4* __restrict__ in, const float* __restrict__ grad,
                                                           int per_row, int64_t N, float4* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float4 r = in[i];
  r.y *= per_row ? grad[i] : grad[0];
  out[i] = r;
}

}  // namespace slf
