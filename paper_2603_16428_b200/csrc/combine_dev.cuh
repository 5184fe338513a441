// combine_dev.cuh — the per-row statistics combine of schedule S with the per-row stash reference
// as a device function of 128 threads, run by the dX+dW group launch's epilogue
// warps before their first tile (DESIGN.md §6 "in-kernel combine"); the same arithmetic, in the
// same order, as combine_scale_kernel (s_kernels.cuh) for a single GPU:
//   lse_i = merge of the row's (m_t, s_t) tile partials (32 lanes, tiles p, p+32, ... per lane,
//           lanes merged in lane order), loss row, RowStat, row factor f_i = coef exp(M_i - lse_i);
//   rows whose per-row reference does not fit are rescaled in place (rare);
//   X'^T[h][i] = bf16(f_i x_ih).
// Plus the synchronisation helpers of the launch: an arrival counter per chunk and an acquire
// spin (bounded: a trap instead of a hang).
#pragma once
#include <cstdint>

#include "../../include/slf_lce.h"
#include "aux_kernels.cuh"
#include "ptx.cuh"

namespace slf {

__device__ __forceinline__ float coef_of(int reduction, float scale, unsigned long long n_valid) {
  return (reduction == SLF_MEAN) ? (n_valid ? scale / (float)n_valid : 0.f) : scale;
}

// A tile whose max exceeds the row reference by more than this keeps its own max in the stash
// (exp(70) = 2.5e30: far from the bf16 / fp32 overflow at exp(88.7)).
constexpr float STASH_REF_SLACK = 70.f;

// Arguments of the in-kernel combine (one chunk; single GPU, per-row reference, no RMSNorm jobs).
struct CombineJob {
  const float2* partials;  // [tiles][rows] (m_t, s_t)
  const float* zt;         // row 0 of the chunk
  const int32_t* t;
  const float* mref;
  const WsHeader* hdr;
  float* loss_rows;
  slf_rowstat* rowstat;
  float* fac;
  uint16_t* stash;   // rows [0, split) (workspace)
  uint16_t* stash2;  // rows [split, rows) (extended stash in dhidden)
  const uint16_t* xrows;
  uint16_t* xs;  // X'^T [H][ld_xst]
  int64_t V_l, ld_stash, H, ld_xst;
  int tiles, rows, split, reduction;
  int32_t ign;
  float scale, grad_scale;
  unsigned* counter;         // arrivals of the launch's CTAs (zeroed per call)
  const unsigned* fb_flag;   // set by the stash epilogue when a row may need the in-place rescale
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Generic-proxy global writes (seen through an acquire) before later async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Wait until *p >= target.  Every CTA of the launch becomes resident (one per SM, persistent; the
// kernels before it finish on their own) and arrives after a bounded amount of work, so this ends;
// a trap after ~30 s (e.g. SMs held that long by other work on the device) turns a stall into a
// launch failure instead of a hung GPU.
__device__ __forceinline__ void spin_until_geq(const unsigned* p, unsigned target) {
  unsigned long long n = 0;
  while (ld_acquire_u32(p) < target) {
    __nanosleep(128);
    if (++n > (1ull << 28)) __trap();
  }
}

constexpr int CJ_ROWS = 4, CJ_LANES = 32, CJ_THREADS = 128;

// The combine rows [4 rg, 4 rg + 4) for rg = first, first + step, ...: 128 threads (tid 0..127, the
// caller's epilogue warps), named barrier `bar`; scratch >= (3 * 32 * 4 + 16) * 4 + tiles * 4 bytes
// of shared memory.
__device__ __noinline__ void combine_rows_dev(const CombineJob& cj, int first, int step, int tid, uint32_t bar,
                                              float* scratch) {
  float(*lm)[CJ_ROWS] = reinterpret_cast<float(*)[CJ_ROWS]>(scratch);
  float(*ls)[CJ_ROWS] = reinterpret_cast<float(*)[CJ_ROWS]>(scratch + CJ_LANES * CJ_ROWS);
  int(*lfb)[CJ_ROWS] = reinterpret_cast<int(*)[CJ_ROWS]>(scratch + 2 * CJ_LANES * CJ_ROWS);
  float* sF = scratch + 3 * CJ_LANES * CJ_ROWS;
  float* sLse = sF + CJ_ROWS;
  float* sCg = sLse + CJ_ROWS;
  int* sFb = reinterpret_cast<int*>(sCg + CJ_ROWS);
  float* r_t = reinterpret_cast<float*>(sFb + CJ_ROWS);  // [tiles]
  const int rows = cj.rows, tiles = cj.tiles;
  const int groups = (rows + CJ_ROWS - 1) / CJ_ROWS;
  const int rl = tid % CJ_ROWS, lane = tid / CJ_ROWS;
  for (int rg = first; rg < groups; rg += step) {
    const int i0 = rg * CJ_ROWS;
    {
      const int i = i0 + rl;
      float m = -INFINITY, sum = 0.f;
      int fb = 0;
      if (i < rows) {
        const float M = cj.mref[i];
#pragma unroll 4
        for (int k = lane; k < tiles; k += CJ_LANES) {
          const float2 p = cj.partials[(size_t)k * rows + i];
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
    named_bar_sync(bar, CJ_THREADS);
    if (tid < CJ_ROWS && i0 + tid < rows) {  // one thread per row: lanes in order
      const int i = i0 + tid;
      float Mx = -INFINITY, S = 0.f;
      int fb = 0;
      for (int p = 0; p < CJ_LANES; ++p) {
        Mx = fmaxf(Mx, lm[p][tid]);
        fb |= lfb[p][tid];
      }
      for (int p = 0; p < CJ_LANES; ++p)
        if (lm[p][tid] != -INFINITY) S += ls[p][tid] * ex2((lm[p][tid] - Mx) * LOG2E);
      const int32_t tt = cj.t[i];
      const bool valid = tt != cj.ign;
      const bool bad = valid && (tt < 0 || (int64_t)tt >= cj.V_l);
      const bool here = valid && !bad;
      const float z = here ? cj.zt[i] : 0.f;
      const float lse = Mx + logf(S);
      const float coef = (valid && !bad) ? coef_of(cj.reduction, cj.scale, cj.hdr->n_valid) : 0.f;
      float l = valid ? (lse - z) : 0.f;
      if (bad) l = __int_as_float(0x7fc00000);
      cj.loss_rows[i] = l;
      cj.rowstat[i] = slf_rowstat{lse * LOG2E, coef, here ? (int32_t)tt : -1, valid ? 1 : 0};
      const float cg = coef * cj.grad_scale;
      float f = 0.f;
      if (cg != 0.f) {
        f = cg * ex2((cj.mref[i] - lse) * LOG2E);
        if (!(fabsf(f) >= 1e-30f && fabsf(f) <= 1e30f)) fb = 1;
      }
      sLse[tid] = lse;
      sCg[tid] = cg;
      sFb[tid] = fb;
      sF[tid] = fb ? 1.f : f;
      cj.fac[i] = fb ? 1.f : f;
    }
    named_bar_sync(bar, CJ_THREADS);
    for (int r = 0; r < CJ_ROWS && i0 + r < rows; ++r) {  // rare: rescale a stash row in place to G_P
      if (!sFb[r]) continue;
      const int i = i0 + r;
      const float M = cj.mref[i], lse = sLse[r], cg = sCg[r];
      for (int k = tid; k < tiles; k += CJ_THREADS) {
        const float mt = cj.partials[(size_t)k * rows + i].x;
        float f;
        if (mt - M > STASH_REF_SLACK) f = cg * ex2((mt - lse) * LOG2E);
        else if (M - mt > 80.f) f = 0.f;
        else f = cg * ex2((M - mt) * LOG2E) * ex2((mt - lse) * LOG2E);
        r_t[k] = f;
      }
      named_bar_sync(bar, CJ_THREADS);
      uint4* row = reinterpret_cast<uint4*>(i < cj.split ? cj.stash + (size_t)i * cj.ld_stash
                                                         : cj.stash2 + (size_t)(i - cj.split) * cj.ld_stash);
      const int64_t q8 = (cj.V_l + 7) / 8;
      for (int64_t q = tid; q < q8; q += CJ_THREADS) {
        const float f = r_t[(q * 8) / 256];
        uint4 x = row[q];
        x.x = pack_bf16x2(bf16lo_to_f32(x.x) * f, bf16hi_to_f32(x.x) * f);
        x.y = pack_bf16x2(bf16lo_to_f32(x.y) * f, bf16hi_to_f32(x.y) * f);
        x.z = pack_bf16x2(bf16lo_to_f32(x.z) * f, bf16hi_to_f32(x.z) * f);
        x.w = pack_bf16x2(bf16lo_to_f32(x.w) * f, bf16hi_to_f32(x.w) * f);
        row[q] = x;
      }
      named_bar_sync(bar, CJ_THREADS);
    }
    // X'^T[h][i0 .. i0 + 4): 8 consecutive columns per thread, four 16-byte row loads, a register
    // transpose, eight 8-byte column stores (f = 1 for rescaled rows: an exact copy)
    const int nr = min(CJ_ROWS, rows - i0);
    if (!cj.xs) {  // no dW GEMM: no X'
    } else if (nr == CJ_ROWS && (cj.H % 8) == 0) {
      for (int64_t h0 = (int64_t)tid * 8; h0 < cj.H; h0 += CJ_THREADS * 8) {
        float v[CJ_ROWS][8];
#pragma unroll
        for (int r = 0; r < CJ_ROWS; ++r) {
          const uint4 q = *reinterpret_cast<const uint4*>(cj.xrows + (size_t)(i0 + r) * cj.H + h0);
          const float f = sF[r];
          v[r][0] = bf16lo_to_f32(q.x) * f; v[r][1] = bf16hi_to_f32(q.x) * f;
          v[r][2] = bf16lo_to_f32(q.y) * f; v[r][3] = bf16hi_to_f32(q.y) * f;
          v[r][4] = bf16lo_to_f32(q.z) * f; v[r][5] = bf16hi_to_f32(q.z) * f;
          v[r][6] = bf16lo_to_f32(q.w) * f; v[r][7] = bf16hi_to_f32(q.w) * f;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint2*>(cj.xs + (size_t)(h0 + c) * cj.ld_xst + i0) =
              make_uint2(pack_bf16x2(v[0][c], v[1][c]), pack_bf16x2(v[2][c], v[3][c]));
      }
    } else {
      for (int64_t h = tid; h < cj.H; h += CJ_THREADS)
        for (int r = 0; r < nr; ++r) {
          const float x = __uint_as_float((uint32_t)cj.xrows[(size_t)(i0 + r) * cj.H + h] << 16) * sF[r];
          cj.xs[(size_t)h * cj.ld_xst + i0 + r] = (uint16_t)(pack_bf16x2(x, 0.f) & 0xFFFFu);
        }
    }
    named_bar_sync(bar, CJ_THREADS);  // the scratch is reused by the next row group
  }
}

}  // namespace slf
