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
// One launch between chunk k-1's grouped dX/dW GEMMs and chunk k's stash GEMM does three disjoint
// jobs, by block index:
//   [0, nb_bwd)                    backward of chunk k-1's rows: dy (bf16, the group's dX output in
//                                  the caller's dx rows) -> dx in place, and this block's fp32 dg
//                                  partial over its rows -> part_b[block][H]
//   [nb_bwd, nb_bwd + f_rows)      forward of chunk k's rows: y = bf16(x * rstd * g) into the chunk
//                                  buffer ybuf (the GEMMs' A / B operand), rstd kept for the backward
//   [.., + nb_red)                 dg += sum_b part_r[b][:] for chunk k-2 (its partials complete:
//                                  an earlier launch), 256 columns per block, block order
// y never exists for all N rows: only the chunk's rows, which stay in L2 between the kernels that
// read them.  Launched with programmatic dependent launch; every block waits for the previous grid.
struct RmsStep {
  const uint16_t* x;
  const uint16_t* g;
  int64_t H;
  float eps;
  float* rstd;  // [N]
  // backward part
  int64_t b_r0, b_rows;
  int b_rpb, nb_bwd;
  uint16_t* dx;  // [N][H]: dy in, dx out (row-owned, in place)
  float* part_b;
  // forward part
  int64_t f_r0, f_rows;
  uint16_t* ybuf;  // [f_rows][H]
  // dg reduction part
  int nb_red, red_nblk, red_first;
  const float* part_r;
  float* dg;
};

__global__ void __launch_bounds__(RMS_THREADS) rms_step_kernel(RmsStep a) {
  griddep_wait();
  __shared__ float red[RMS_THREADS / 32];
  extern __shared__ float dg_acc[];
  const int64_t groups = a.H / 8;
  const uint4* gr = reinterpret_cast<const uint4*>(a.g);
  int b = blockIdx.x;
  if (b < a.nb_bwd) {  // backward rows [b_r0 + b*rpb, ...)
    for (int64_t j = threadIdx.x; j < a.H; j += RMS_THREADS) dg_acc[j] = 0.f;
    __syncthreads();
    const int64_t r0 = a.b_r0 + (int64_t)b * a.b_rpb, r1 = min(r0 + a.b_rpb, a.b_r0 + a.b_rows);
    for (int64_t row = r0; row < r1; ++row) {
      const float r = a.rstd[row];
      const uint4* xr = reinterpret_cast<const uint4*>(a.x + row * a.H);
      const uint4* dr = reinterpret_cast<const uint4*>(a.dx + row * a.H);
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
          dg_acc[q * 8 + e] += d[e] * xh;
        }
      }
      const float c = block_sum_256(dot, red) / (float)a.H;
      uint4* xo = reinterpret_cast<uint4*>(a.dx + row * a.H);
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
    for (int64_t j = threadIdx.x; j < a.H; j += RMS_THREADS) a.part_b[(size_t)b * a.H + j] = dg_acc[j];
    return;
  }
  b -= a.nb_bwd;
  if (b < a.f_rows) {  // forward row f_r0 + b
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
    uint4* yr = reinterpret_cast<uint4*>(a.ybuf + (int64_t)b * a.H);
    for (int64_t q = threadIdx.x; q < groups; q += RMS_THREADS) {
      float f[8], w[8];
      unpack8(xr[q], f);
      unpack8(gr[q], w);
      yr[q] = make_uint4(pack_bf16x2(f[0] * r * w[0], f[1] * r * w[1]), pack_bf16x2(f[2] * r * w[2], f[3] * r * w[3]),
                         pack_bf16x2(f[4] * r * w[4], f[5] * r * w[5]), pack_bf16x2(f[6] * r * w[6], f[7] * r * w[7]));
    }
    return;
  }
  b -= (int)a.f_rows;
  const int64_t j = (int64_t)b * RMS_THREADS + threadIdx.x;  // dg reduction: column j
  if (j >= a.H) return;
  float sum = 0.f;
  for (int k = 0; k < a.red_nblk; ++k) sum += a.part_r[(size_t)k * a.H + j];
  a.dg[j] = a.red_first ? sum : a.dg[j] + sum;
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

}  // namespace slf
