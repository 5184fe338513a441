// gemm.cuh — persistent, warp-specialised TMA -> tcgen05 -> TMEM GEMM core for sm_100a with the
// LCE epilogues fused into the tile.
//
//   D[M, N] = A[M, K] * B[K, N]   (bf16 in, fp32 accumulate in TMEM)
//   A is K-major (stored [M][K]) or MN-major (stored [K][M]); B is K-major (stored [N][K]) or
//   MN-major (stored [K][N]).  One CTA per SM, 128 x 256 output tile, K-step 64 (one 128-byte
//   swizzle row), 4-stage smem ring fed by TMA, two 256-column TMEM accumulators so the epilogue
//   of tile i overlaps the mainloop of tile i+1.
//   warp 0: TMA producer (one lane) | warp 1: tcgen05.mma issuer (one lane) | warp 2: TMEM
//   allocator | warps 4-7: epilogue, thread = accumulator row (TMEM lane).
//
// Epilogues ("fuses the projection and loss calculation, computing gradients in
// small chunks"):
//   EPI_STATS : per (row, 256-column vocab tile) max m and sum exp(z - m); gathers the target logit.
//   EPI_GRAD  : G = coef * (exp(z - lse) - [v == t]) in fp32, rounded to bf16, stored to the chunk.
//   EPI_DW    : dW tile (bf16), store or fp32 read-add-write of the previous partial, through
//               TMA-staged 64-column chunks (epilogue_dw_tma).
//   EPI_DX    : dX tile: fp32 store / accumulate across vocab chunks, final bf16 conversion with
//               ignored rows forced to +0.
//   EPI_F32   : plain fp32 store (test entry point).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "ptx.cuh"
#include "combine_dev.cuh"
#include "../../include/slf_lce.h"

namespace slf {

constexpr int BM = 128;  // accumulator rows per CTA (TMEM lanes)
constexpr int BN = 256;  // accumulator columns (one tcgen05.mma N)
constexpr int BK = 64;   // one 128-byte swizzle row of bf16
constexpr int GEMM_THREADS = 256;

constexpr uint32_t TMEM_COLS = 512;  // 2 x 256-column fp32 accumulators

// CG = 1: one CTA computes a 128 x 256 tile (cta_group::1).  CG = 2: a CTA pair (cluster of 2)
// computes a 256 x 256 tile with cta_group::2 — each CTA stages its own 128 rows of A and half
// (128 rows) of B, the leader issues the MMA, both CTAs hold 128 accumulator rows in TMEM.
// NB = number of 16 KB epilogue staging buffers.  CTA pairs: NB = 2 leaves room for a 6-stage
// operand ring (faster mainloop; the stash and dX launches), NB = 4 for 5 stages (the dW
// read-modify-write epilogue keeps all four old-value chunks in flight).  Both fit 227 KB.
template <int CG, int NB>
struct Cfg {
  static constexpr int TILE_M = BM * CG;
  static constexpr int B_ROWS = BN / CG;  // rows of B (N extent) staged per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = CG == 2 ? (NB <= 2 ? 6 : 5) : 3;
  static constexpr int STAGING_BYTES = NB * BM * 64 * 2;  // [128 rows x 64 bf16] TMA buffers
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGING_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
};

enum EpiKind { EPI_STATS = 0, EPI_GRAD = 1, EPI_DW = 2, EPI_DX = 3, EPI_F32 = 4, EPI_STASH = 5, EPI_DXS = 6 };

// DX epilogue modes (schedule R).
enum DxMode { DX_STORE_F32 = 0, DX_ACC_F32 = 1, DX_ACC_FINAL_BF16 = 2, DX_STORE_FINAL_BF16 = 3 };

struct GemmArgs {
  int M, N, K;
  int tiles_m, tiles_n, num_tiles, group_m;
  // EPI_STATS / EPI_STASH
  const int32_t* targets;  // row 0 of the GEMM
  int64_t tcol0;           // target id that maps to GEMM column 0 (vocab_start + chunk start)
  int32_t ignore_index;
  float2* partials;        // [tiles_n][M]
  float* zt;               // [M]
  // EPI_GRAD / EPI_DX / EPI_DXS
  const slf_rowstat* rowstat;  // row 0 of the GEMM
  int64_t col0;                // chunk start relative to the shard (GRAD: compare with rowstat.tloc)
  float grad_scale;
  int rows_buf;                // GRAD: rows [M, rows_buf) of the G buffer are written as zeros
  const uint16_t* wrow;        // DXS: the shard's W (one-hot gather W[tloc]); row stride ld_w
  int64_t ld_w;
  // outputs
  void* out;
  int64_t ld_out;
  int mode;
  int tma_out;  // EPI_STASH: write the stash through the output tensor map (TMA-staged stores)
  void* out2;  // DX final bf16 destination (row 0 of the GEMM)
  int64_t ld_out2;
  // Schedule S with a per-row stash reference: EPI_STASH stores exp(z - mref[r])
  // instead of exp(z - m_tile) wherever m_tile - mref[r] <= STASH_REF_SLACK (else the tile keeps its
  // own max); EPI_DXS multiplies the row's accumulator by fac[r].  Null: per-tile max / factor 1.
  const float* mref;
  const float* fac;
  // EPI_STASH of a chunk whose combine runs inside the group launch (CombineJob): *fb_flag := 1 when
  // a row of the tile may need the combine's in-place rescale (its dX tiles then wait for it)
  unsigned* fb_flag;
  const WsHeader* fb_hdr;
  int fb_red;
  float fb_scale, fb_gscale;
};

__device__ __forceinline__ void tile_coords(int tile, const GemmArgs& a, int& m_blk, int& n_blk) {
  // Grouped raster: walk group_m row tiles down before stepping to the next column tile, so one
  // wave of tiles shares a few A row-panels and B column-panels in L2.
  const int per_group = a.group_m * a.tiles_n;
  const int g = tile / per_group;
  const int first_m = g * a.group_m;
  const int gm = min(a.group_m, a.tiles_m - first_m);
  const int in = tile - g * per_group;
  m_blk = first_m + in % gm;
  n_blk = in / gm;
}

template <int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& a, uint32_t taddr, int row0, int n_blk, int row_in_tile) {
  const int r = row0 + row_in_tile;
  const bool row_ok = r < a.M;
  const int n0 = n_blk * BN;
  const int ncols = min(BN, a.N - n0);
  uint32_t v[32];

  if constexpr (EPI == EPI_STATS) {
    int tl = -1;
    if (row_ok) {
      const int32_t t = a.targets[r];
      const int64_t loc = (int64_t)t - a.tcol0 - n0;
      tl = (t != a.ignore_index && loc >= 0 && loc < ncols) ? (int)loc : -1;
    }
    float mx = -INFINITY;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;  // warp-uniform
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (c * 32 + i < ncols) mx = fmaxf(mx, __uint_as_float(v[i]));
    }
    const float mb = mx * LOG2E;
    float s = 0.f, zt = 0.f;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float z = __uint_as_float(v[i]);
        const float e = ex2(fmaf(z, LOG2E, -mb));
        s += (c * 32 + i < ncols) ? e : 0.f;
        zt = (c * 32 + i == tl) ? z : zt;
      }
    }
    if (row_ok) {
      a.partials[(size_t)n_blk * a.M + r] = make_float2(mx, s);
      if (tl >= 0) a.zt[r] = zt;
    }
  } else if constexpr (EPI == EPI_STASH) {
    // Schedule S forward: (m, s) per (row, tile) as EPI_STATS, plus the bf16 stash
    // p~ = exp(z - m_tile) of the whole tile (no recompute later).
    int tl = -1;
    if (row_ok) {
      const int32_t t = a.targets[r];
      const int64_t loc = (int64_t)t - a.tcol0 - n0;
      tl = (t != a.ignore_index && loc >= 0 && loc < ncols) ? (int)loc : -1;
    }
    float mx = -INFINITY;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (c * 32 + i < ncols) mx = fmaxf(mx, __uint_as_float(v[i]));
    }
    const float mb = mx * LOG2E;
    float cmul = 1.f;  // stash relative to the row reference: exp(z - m) * exp(m - mref)
    if (a.mref && row_ok) {
      const float M = a.mref[r];
      if (!(mx - M > STASH_REF_SLACK)) cmul = ex2((mx - M) * LOG2E);
    }
    float s = 0.f, zt = 0.f;
    uint16_t* out = reinterpret_cast<uint16_t*>(a.out) + (size_t)r * a.ld_out + n0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
      uint32_t p[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float z0 = __uint_as_float(v[i]), z1 = __uint_as_float(v[i + 1]);
        float e0 = ex2(fmaf(z0, LOG2E, -mb)), e1 = ex2(fmaf(z1, LOG2E, -mb));
        e0 = (c * 32 + i < ncols) ? e0 : 0.f;
        e1 = (c * 32 + i + 1 < ncols) ? e1 : 0.f;
        s += e0 + e1;
        zt = (c * 32 + i == tl) ? z0 : zt;
        zt = (c * 32 + i + 1 == tl) ? z1 : zt;
        p[i / 2] = pack_bf16x2(e0 * cmul, e1 * cmul);
      }
      if (row_ok && !(a.mode & 32)) {  // mode bit 32: skip the stash stores (timing experiment only)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (c * 32 + q * 8 < ncols)
            *reinterpret_cast<uint4*>(out + c * 32 + q * 8) = make_uint4(p[4 * q], p[4 * q + 1], p[4 * q + 2], p[4 * q + 3]);
      }
    }
    if (row_ok) {
      a.partials[(size_t)n_blk * a.M + r] = make_float2(mx, s);
      if (tl >= 0) a.zt[r] = zt;
    }
  } else if constexpr (EPI == EPI_DXS) {
    // Schedule S dX: acc = G_P W (softmax term); subtract the one-hot term coef * W[t] exactly in
    // fp32 (only for targets inside this shard); ignored rows are +0.0.
    float coef = 0.f;
    int tl = -1;
    bool valid = false;
    if (row_ok) {
      const slf_rowstat rs = a.rowstat[r];
      coef = rs.coef * a.grad_scale;
      tl = rs.tloc;
      valid = rs.valid != 0;
    }
    const uint16_t* wt = a.wrow + (size_t)(tl >= 0 ? tl : 0) * a.ld_w + n0;
    const float fr = (a.fac && row_ok) ? a.fac[r] : 1.f;  // per-row stash reference factor
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
      if (row_ok) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = c * 32 + q * 8;
          if (j < ncols) {
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[q * 8 + e]) * fr;
            if (tl >= 0) {
              const uint4 w = *reinterpret_cast<const uint4*>(wt + j);
              f[0] -= coef * bf16lo_to_f32(w.x); f[1] -= coef * bf16hi_to_f32(w.x);
              f[2] -= coef * bf16lo_to_f32(w.y); f[3] -= coef * bf16hi_to_f32(w.y);
              f[4] -= coef * bf16lo_to_f32(w.z); f[5] -= coef * bf16hi_to_f32(w.z);
              f[6] -= coef * bf16lo_to_f32(w.w); f[7] -= coef * bf16hi_to_f32(w.w);
            }
            if (!valid)
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] = 0.f;
            if (a.mode == 0) {
              uint16_t* o = reinterpret_cast<uint16_t*>(a.out) + (size_t)r * a.ld_out + n0 + j;
              *reinterpret_cast<uint4*>(o) = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                                                        pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
            } else {
              float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (size_t)r * a.ld_out + n0 + j);
              o[0] = make_float4(f[0], f[1], f[2], f[3]);
              o[1] = make_float4(f[4], f[5], f[6], f[7]);
            }
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_GRAD) {
    float coef = 0.f, lse2 = 0.f;
    int tl = -1;
    if (row_ok) {
      const slf_rowstat rs = a.rowstat[r];
      coef = rs.coef * a.grad_scale;
      lse2 = rs.lse2;
      const int64_t loc = (int64_t)rs.tloc - a.col0 - n0;
      tl = (rs.tloc >= 0 && loc >= 0 && loc < ncols) ? (int)loc : -1;
    }
    uint16_t* out = reinterpret_cast<uint16_t*>(a.out) + (size_t)r * a.ld_out + n0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
      uint32_t p[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const int j0 = c * 32 + i, j1 = j0 + 1;
        float g0 = coef * ex2(fmaf(__uint_as_float(v[i]), LOG2E, -lse2)) - (j0 == tl ? coef : 0.f);
        float g1 = coef * ex2(fmaf(__uint_as_float(v[i + 1]), LOG2E, -lse2)) - (j1 == tl ? coef : 0.f);
        g0 = j0 < ncols ? g0 : 0.f;
        g1 = j1 < ncols ? g1 : 0.f;
        p[i / 2] = pack_bf16x2(g0, g1);
      }
      if (r < a.rows_buf) {  // rows past M (inside the buffer) are written as zeros
        uint4* dst = reinterpret_cast<uint4*>(out + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = row_ok ? make_uint4(p[4 * q], p[4 * q + 1], p[4 * q + 2], p[4 * q + 3]) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
  } else if constexpr (EPI == EPI_DX) {
    const bool valid = row_ok && a.rowstat[r].valid != 0;
    float* acc = reinterpret_cast<float*>(a.out) + (size_t)r * a.ld_out + n0;
    uint16_t* fin = reinterpret_cast<uint16_t*>(a.out2) + (size_t)r * a.ld_out2 + n0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
      if (row_ok) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = c * 32 + q * 8;
          if (j < ncols) {
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = valid ? __uint_as_float(v[q * 8 + e]) : 0.f;
            float4* d4 = reinterpret_cast<float4*>(acc + j);
            if (a.mode == DX_ACC_F32 || a.mode == DX_ACC_FINAL_BF16) {
              const float4 o0 = d4[0], o1 = d4[1];
              f[0] += o0.x; f[1] += o0.y; f[2] += o0.z; f[3] += o0.w;
              f[4] += o1.x; f[5] += o1.y; f[6] += o1.z; f[7] += o1.w;
            }
            if (a.mode == DX_STORE_F32 || a.mode == DX_ACC_F32) {
              d4[0] = make_float4(f[0], f[1], f[2], f[3]);
              d4[1] = make_float4(f[4], f[5], f[6], f[7]);
            } else {
              uint4 o = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                   pack_bf16x2(f[6], f[7]));
              if (!valid) o = make_uint4(0u, 0u, 0u, 0u);  // +0.0 exactly for ignored rows
              *reinterpret_cast<uint4*>(fin + j) = o;
            }
          }
        }
      }
    }
  } else {  // EPI_F32
    float* out = reinterpret_cast<float*>(a.out) + (size_t)r * a.ld_out + n0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      if (c * 32 >= ncols) break;
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
      if (row_ok) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c * 32 + i < ncols) out[c * 32 + i] = __uint_as_float(v[i]);
      }
    }
  }
}

// dW tile epilogue through TMA (store, or read-add-write of the previous bf16 partial when
// mode == 1).  The 128 x 256 tile is split into four 64-column chunks, one swizzled 16 KB smem
// buffer each.  The old chunks are requested by TMA (coalesced) BEFORE the accumulator is waited
// for, so their latency hides behind this tile's MMAs; each thread then adds its row's fp32
// accumulator from TMEM, writes bf16 back to smem, and four TMA stores write the tile out.
// Thread-per-row global accesses would touch 32 cache lines per warp instruction; this keeps the
// short-K dW GEMMs of schedule S tensor-bound instead of epilogue-bound.
template <int NB, typename WaitAcc, typename ReleaseTmem>
__device__ __forceinline__ void epilogue_dw_tma(const GemmArgs& a, const CUtensorMap* tmC, uint32_t taddr, int row0,
                                                int n_blk, int rl, uint8_t* stg, uint64_t* sbar, uint32_t& sphase,
                                                uint32_t& sq, bool lead, WaitAcc wait_acc, ReleaseTmem release_tmem,
                                                int dbg = 0) {
  constexpr uint32_t CHUNK_BYTES = BM * 64 * 2;
  // chunks are processed NB at a time through the NB staging buffers
  const int n0 = n_blk * BN;
  const int nch = min(BN, a.N - n0 + 63) / 64;  // 64-column chunks with at least one valid column
  const bool rmw = a.mode == 1;
  const uint32_t sbase = smem_u32(stg);
  if (!rmw && !(dbg & 1024)) {
    // Store / L2 reduce-add (no old values): pull the whole 256-column accumulator row into
    // registers as bf16 pairs (128 registers) and hand TMEM back to the MMA issuer at once; the
    // staging-buffer waits on earlier TMA stores then only delay these warps, never the next
    // tile's MMAs (they have a whole mainloop to finish).
    uint32_t pk[BN / 2];
    wait_acc();
#pragma unroll
    for (int k = 0; k < BN / 64; ++k) {
      uint32_t w0[32], w1[32];
      if (k < nch) {
        tmem_ld32(taddr + k * 64, w0);
        tmem_ld32(taddr + k * 64 + 32, w1);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          pk[k * 32 + e] = pack_bf16x2(__uint_as_float(w0[2 * e]), __uint_as_float(w0[2 * e + 1]));
          pk[k * 32 + 16 + e] = pack_bf16x2(__uint_as_float(w1[2 * e]), __uint_as_float(w1[2 * e + 1]));
        }
      }
    }
    release_tmem();
    if (!(dbg & 4096)) {
      // Chunk-pipelined staging: one bulk group per 64-column chunk, buffers used round-robin by a
      // sequence number that runs on across tiles (sq), and before refilling a buffer only the store
      // that last read it must be done (at most NB-1 newer groups pending) — the TMA reads chunk k
      // while the warps fill chunk k+1, instead of NB chunks filled, stored, and all waited for.
#pragma unroll
      for (int k = 0; k < BN / 64; ++k) {
        if (k >= nch) break;
        const int j = (int)(sq % NB);
        if (lead) bulk_wait_read<NB - 1>();
        named_bar_sync(1, 128);
        const uint32_t rowaddr = sbase + j * CHUNK_BYTES + rl * 128;
#pragma unroll
        for (int gi = 0; gi < 8; ++gi) {
          const uint32_t* src = &pk[k * 32 + gi * 4];
          sts128(rowaddr + ((gi ^ (rl & 7)) << 4), make_uint4(src[0], src[1], src[2], src[3]));
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (lead) {
          if (dbg & 256) {
            // timing experiment only: no dW store at all (wrong dW)
          } else if (a.mode == 2) {
            tma_reduce_add_2d(tmC, stg + j * CHUNK_BYTES, n0 + k * 64, row0);
          } else {
            tma_store_2d(tmC, stg + j * CHUNK_BYTES, n0 + k * 64, row0);
          }
          bulk_commit();
        }
        ++sq;
      }
      return;
    }
#pragma unroll
    for (int g0 = 0; g0 < BN / 64; g0 += NB) {
      if (g0 >= nch) break;
      const int gn = min(NB, nch - g0);
      if (lead) bulk_wait_read<0>();  // the previous stores have read the staging buffers
      named_bar_sync(1, 128);
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (j < gn) {
          const uint32_t rowaddr = sbase + j * CHUNK_BYTES + rl * 128;
#pragma unroll
          for (int gi = 0; gi < 8; ++gi) {
            const uint32_t* src = &pk[(g0 + j) * 32 + gi * 4];
            sts128(rowaddr + ((gi ^ (rl & 7)) << 4), make_uint4(src[0], src[1], src[2], src[3]));
          }
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (lead) {
        if (dbg & 256) {
          // timing experiment only: no dW store at all (wrong dW)
        } else if (a.mode == 2) {
          for (int j = 0; j < gn; ++j) tma_reduce_add_2d(tmC, stg + j * CHUNK_BYTES, n0 + (g0 + j) * 64, row0);
        } else {
          for (int j = 0; j < gn; ++j) tma_store_2d(tmC, stg + j * CHUNK_BYTES, n0 + (g0 + j) * 64, row0);
        }
        bulk_commit();
      }
    }
    return;
  }
  uint32_t v0[32], v1[32];
  for (int g0 = 0; g0 < nch; g0 += NB) {
    const int gn = min(NB, nch - g0);
    // The previous stores (of the last tile, or of the previous group) must have read the buffers.
    if (lead) bulk_wait_read<0>();
    named_bar_sync(1, 128);
    if (g0 == 0 && (dbg & 2)) wait_acc();
    if (rmw && lead) {
      for (int j = 0; j < gn; ++j) {
        mbar_arrive_expect_tx(&sbar[j], CHUNK_BYTES);
        tma_load_2d(tmC, &sbar[j], stg + j * CHUNK_BYTES, n0 + (g0 + j) * 64, (dbg & 32) ? (row0 & 1023) : row0,
                    (dbg & 16) ? policy_evict_first() : policy_evict_normal());
      }
    }
    if (g0 == 0 && !(dbg & 2)) wait_acc();
    for (int j = 0; j < gn; ++j) {
      const int k = g0 + j;
      tmem_ld32(taddr + k * 64, v0);
      tmem_ld32(taddr + k * 64 + 32, v1);
      tmem_ld_wait();
      if (k == nch - 1) release_tmem();  // the accumulator is in registers: let the next MMA start
      if (rmw) {
        mbar_wait(&sbar[j], (sphase >> j) & 1);
        sphase ^= 1u << j;
      }
      const uint32_t rowaddr = sbase + j * CHUNK_BYTES + rl * 128;
#pragma unroll
      for (int gi = 0; gi < 8; ++gi) {
        const uint32_t addr = rowaddr + ((gi ^ (rl & 7)) << 4);  // 128B swizzle: granule gi of row rl
        const uint32_t* src = gi < 4 ? &v0[gi * 8] : &v1[(gi - 4) * 8];
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(src[e]);
        if (rmw) {
          const uint4 o = lds128(addr);
          f[0] += bf16lo_to_f32(o.x); f[1] += bf16hi_to_f32(o.x);
          f[2] += bf16lo_to_f32(o.y); f[3] += bf16hi_to_f32(o.y);
          f[4] += bf16lo_to_f32(o.z); f[5] += bf16hi_to_f32(o.z);
          f[6] += bf16lo_to_f32(o.w); f[7] += bf16hi_to_f32(o.w);
        }
        sts128(addr, make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                pack_bf16x2(f[6], f[7])));
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (lead) {
      if (dbg & 256) {
        // timing experiment only: no dW store at all (wrong dW)
      } else if (a.mode == 2) {  // accumulate in L2: bf16 reduce-add of this tile's partial
        for (int j = 0; j < gn; ++j) tma_reduce_add_2d(tmC, stg + j * CHUNK_BYTES, n0 + (g0 + j) * 64, row0);
      } else if (dbg & 16) {
        const uint64_t pol = policy_evict_first();
        for (int j = 0; j < gn; ++j) tma_store_2d_hint(tmC, stg + j * CHUNK_BYTES, n0 + (g0 + j) * 64, row0, pol);
      } else {
        for (int j = 0; j < gn; ++j) tma_store_2d(tmC, stg + j * CHUNK_BYTES, n0 + (g0 + j) * 64, row0);
      }
      bulk_commit();
    }
  }
}

// Schedule S forward epilogue with TMA-staged stash stores: per (row, 256-column tile) the max m_t
// and sum exp(z - m_t) (as EPI_STATS), the target-logit gather, and the bf16 stash
// p~ = exp(z - m_t) written through four swizzled 16 KB smem chunks and TMA stores (coalesced),
// instead of thread-per-row 16-byte stores that touch 32 cache lines per warp instruction.
template <int NB, typename WaitAcc, typename ReleaseTmem>
__device__ __forceinline__ void epilogue_stash_tma(const GemmArgs& a, const CUtensorMap* tmC, uint32_t taddr,
                                                   int row0, int n_blk, int rl, uint8_t* stg, bool lead,
                                                   WaitAcc wait_acc, ReleaseTmem release_tmem, uint32_t& sq,
                                                   int c_off = 0) {
  constexpr uint32_t CHUNK_BYTES = BM * 64 * 2;
  const int r = row0 + rl;
  const bool row_ok = r < a.M;
  const int n0 = n_blk * BN;
  const int ncols = min(BN, a.N - n0);
  const uint32_t sbase = smem_u32(stg);
  int tl = -1;
  if (row_ok) {
    const int32_t t = a.targets[r];
    const int64_t loc = (int64_t)t - a.tcol0 - n0;
    tl = (t != a.ignore_index && loc >= 0 && loc < ncols) ? (int)loc : -1;
  }
  wait_acc();
  uint32_t v[32];
  float mx = -INFINITY;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    if (c * 32 >= ncols) break;
    tmem_ld32(taddr + c * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c * 32 + i < ncols) mx = fmaxf(mx, __uint_as_float(v[i]));
  }
  const float mb = mx * LOG2E;
  float cmul = 1.f;  // stash relative to the row reference: exp(z - m) * exp(m - mref)
  if (a.mref && row_ok) {
    const float M = a.mref[r];
    if (!(mx - M > STASH_REF_SLACK)) cmul = ex2((mx - M) * LOG2E);
    if (a.fb_flag) {
      // In-kernel combine (CombineJob): the group's dX tiles read this stash before the combine ran,
      // which is only right if no row needs its in-place rescale.  A row may need it when a tile
      // kept its own max (mx - M > SLACK) or when f = cg exp(M - lse) can leave [1e-30, 1e30]:
      // M - lse <= M - z_t = STASH_REF_SHIFT (40) bounds it above; lse <= max_t m_t + ln V bounds it
      // below, so f >= 1e-30 (with a factor e of margin) while mx - M <= ln|cg| + 68 - ln V.
      float lim = STASH_REF_SLACK;
      const float cg = fabsf(coef_of(a.fb_red, a.fb_scale, a.fb_hdr->n_valid) * a.fb_gscale);
      if (cg != 0.f) {
        if (!(cg * 2.36e17f <= 1e29f)) lim = -INFINITY;
        else lim = fminf(lim, __logf(cg) + 68.f - __logf((float)a.N));
      }
      if (!(mx - M <= lim)) atomicOr(a.fb_flag, 1u);
    }
  }
  // Per 64-column chunk: two 32-column TMEM loads -> exp -> bf16 pairs -> one staging buffer ->
  // one TMA store, chunk-pipelined as the dW epilogue: one bulk group per chunk, buffers by a running
  // sequence, a buffer is refilled once the store that last read it is done.  TMEM is released
  // after the last load.
  float s = 0.f, zt = 0.f;
  const int nch = (ncols + 63) / 64;
#pragma unroll 1
  for (int k = 0; k < BN / 64; ++k) {
    if (k >= nch) break;
    uint32_t p[32];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * k + h;
      if (c * 32 < ncols) {
        tmem_ld32(taddr + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float z0 = __uint_as_float(v[i]), z1 = __uint_as_float(v[i + 1]);
          float e0 = ex2(fmaf(z0, LOG2E, -mb)), e1 = ex2(fmaf(z1, LOG2E, -mb));
          e0 = (c * 32 + i < ncols) ? e0 : 0.f;
          e1 = (c * 32 + i + 1 < ncols) ? e1 : 0.f;
          s += e0 + e1;
          zt = (c * 32 + i == tl) ? z0 : zt;
          zt = (c * 32 + i + 1 == tl) ? z1 : zt;
          p[h * 16 + i / 2] = pack_bf16x2(e0 * cmul, e1 * cmul);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) p[h * 16 + i] = 0u;
      }
    }
    if (k == nch - 1) release_tmem();
    const int j = (int)(sq % NB);
    if (lead) bulk_wait_read<NB - 1>();
    named_bar_sync(1, 128);
    const uint32_t rowaddr = sbase + j * CHUNK_BYTES + rl * 128;
#pragma unroll
    for (int gi = 0; gi < 8; ++gi)
      sts128(rowaddr + ((gi ^ (rl & 7)) << 4), make_uint4(p[gi * 4], p[gi * 4 + 1], p[gi * 4 + 2], p[gi * 4 + 3]));
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (lead) {
      if (!(a.mode & 32)) tma_store_2d(tmC, stg + j * CHUNK_BYTES, n0 + k * 64, row0 - c_off);  // 32: timing only
      bulk_commit();
    }
    ++sq;
  }
  if (row_ok) {
    a.partials[(size_t)n_blk * a.M + r] = make_float2(mx, s);
    if (tl >= 0) a.zt[r] = zt;
  }
}

// Runtime epilogue dispatch (one problem of a group decides per tile).
__device__ __forceinline__ void epilogue_dispatch(int epi, const GemmArgs& a, uint32_t taddr, int row0, int n_blk,
                                                  int row_in_tile) {
  switch (epi) {
    case EPI_STATS: epilogue_tile<EPI_STATS>(a, taddr, row0, n_blk, row_in_tile); break;
    case EPI_GRAD: epilogue_tile<EPI_GRAD>(a, taddr, row0, n_blk, row_in_tile); break;
    case EPI_DX: epilogue_tile<EPI_DX>(a, taddr, row0, n_blk, row_in_tile); break;
    case EPI_STASH: epilogue_tile<EPI_STASH>(a, taddr, row0, n_blk, row_in_tile); break;
    case EPI_DXS: epilogue_tile<EPI_DXS>(a, taddr, row0, n_blk, row_in_tile); break;
    default: epilogue_tile<EPI_F32>(a, taddr, row0, n_blk, row_in_tile); break;
  }
}

// ---- grouped persistent kernel ---------------------------------------------------------------
// Up to MAXP independent GEMM problems share one launch (e.g. the dW and dX GEMMs of one chunk):
// problem p owns global tiles [tile_begin[p], tile_begin[p+1]).  Each unit (CTA or CTA pair) walks
// either a host-built list (sched: balanced by K-blocks, longest first) or tiles u, u+units, ...
constexpr int MAXP = 2;

// Debug trace (slf_debug_trace_read): per-tile clock64 stamps of unit 0's leader CTA for one
// selected launch.  Slots per tile: 0 MMA before tempty wait, 1 after it, 2 MMA tile issued,
// 3 epilogue start, 4 accumulator ready, 5 TMEM released, 6 epilogue end, 7 problem index.
// After the tile slots, per unit (leader CTA), when tracing: 0 MMA cycles waiting on full stages,
// 1 MMA cycles waiting on a free accumulator, 2 first MMA-loop clock, 3 last, 4 K-blocks issued,
// 5 producer cycles waiting on empty stages, 6 tiles, 7 globaltimer ns from first to last clock.
constexpr int TRACE_TILES = 1024;
constexpr int TRACE_UNITS = 256;
__device__ unsigned long long g_trace[TRACE_TILES * 8 + TRACE_UNITS * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long clk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

// A problem's A operand (and the TMA-staged output C) may live in two row segments of different
// tensors (schedule S's stash extended into the caller's free dhidden rows): rows (the tensor's
// outer dimension) >= a_split come from map A2 at row - a_split, output rows >= c_split go to C2.
constexpr int MAPS_PER_PROB = 5;  // A, B, C, A2, C2
constexpr int NO_SPLIT = 0x7fffffff;

struct Prob {
  GemmArgs a;
  int epi, a_mn, b_mn, tile_begin;
  int a_split, c_split;
  int a3d, b3d;  // MN-major operand maps are 3-D {64, K, MN/64}: one TMA box per stage
};

struct GroupArgs {
  Prob p[MAXP];
  int nprob;
  int num_tiles;
  int dbg;  // timing-experiment knobs (0 in production): 1 = no L2 prefetch, 2 = late old-dW loads,
            // 4 = record the per-tile trace of unit 0, 8 = L2 prefetch of the next tile's MN-major A,
            // 16 = evict-first dW RMW traffic, 32 = old-dW loads from the first 1024 rows (wrong dW),
            // 256 = no dW stores (wrong dW), 1024 = dW epilogue in the old order (TMEM held until the
            // staging buffers are free), 2048 = MN-major A operands read from two K-blocks only (wrong)
  const int* sched;  // [units][sched_stride] tile ids, -1 terminated (nullptr: round robin)
  int sched_stride;
  // il = 1: the table holds (tile, seg) int pairs — a K-block range [kb0, kb1) of the tile, whether it
  // starts / ends the tile's accumulation, and its TMEM accumulator slot (the dX tiles
  // split into K segments interleaved with the dW tiles of the same vocabulary range)
  int il;
  // early = 1: the operands are call inputs no kernel writes (the stash GEMM's hidden rows and W),
  // so the TMA producer and the MMA issuer start while the previous grid drains (PDL); every other
  // warp, the epilogue among them, waits for it before any global access
  int early;
  // cj_on = 1: the chunk's per-row combine runs here: the epilogue warps of every CTA
  // combine their share of rows first and arrive on cj.counter; the producer waits for all arrivals
  // before the first dW tile (X'^T) — and before anything when the stash flagged a rescale — and the
  // epilogues before their first tile (RowStat, row factors)
  int cj_on;
  CombineJob cj;
};

// One work item of a unit: a whole tile (il = 0), or a K segment of one (il = 1).
struct Item {
  int tile, kb0, kb1, first, last, slot;  // slot -1: alternate accumulators by tile (il = 0)
};

struct TMaps {
  CUtensorMap m[MAPS_PER_PROB * MAXP];  // A, B, C (TMA-staged output), A2, C2 of each problem
};

struct TileIter {
  const GroupArgs& g;
  int unit, units, i;
  __device__ TileIter(const GroupArgs& g_, int unit_, int units_) : g(g_), unit(unit_), units(units_), i(0) {}
  __device__ __forceinline__ int at(int k) const {
    int t;
    if (g.sched) {
      t = k < g.sched_stride ? __ldg(g.sched + (size_t)unit * g.sched_stride + k) : -1;
    } else {
      t = unit + k * units;
      if (t >= g.num_tiles) t = -1;
    }
    return t;
  }
  __device__ __forceinline__ int next() { return at(i++); }
  __device__ __forceinline__ int peek() const {
    if (!g.il) return at(i);
    return 2 * i < g.sched_stride ? __ldg(g.sched + (size_t)unit * g.sched_stride + 2 * i) : -1;
  }
  __device__ __forceinline__ Item next_item() {
    Item r;
    if (!g.il) {
      r.tile = at(i++);
      r.kb0 = 0;
      r.kb1 = 0;  // the caller's problem K
      r.first = r.last = 1;
      r.slot = -1;
      return r;
    }
    const int k = i++;
    r.tile = 2 * k < g.sched_stride ? __ldg(g.sched + (size_t)unit * g.sched_stride + 2 * k) : -1;
    const int sg = r.tile >= 0 ? __ldg(g.sched + (size_t)unit * g.sched_stride + 2 * k + 1) : 0;
    r.kb0 = sg & 4095;
    r.kb1 = (sg >> 12) & 4095;
    r.first = (sg >> 24) & 1;
    r.last = (sg >> 25) & 1;
    r.slot = (sg >> 26) & 1;
    return r;
  }
};

__device__ __forceinline__ int prob_of(const GroupArgs& g, int tile) {
  return (g.nprob > 1 && tile >= g.p[1].tile_begin) ? 1 : 0;
}

template <int CG, int NB>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    lce_group_kernel(const __grid_constant__ TMaps tm, const __grid_constant__ GroupArgs g) {
  using C = Cfg<CG, NB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* stg = smem + C::STAGES * C::STAGE_BYTES;  // NB x 16 KB epilogue staging (1024-aligned)
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + C::STAGING_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sbar = tempty + 2;  // staging-load barriers (4)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sbar + 4);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // 0 = pair leader
  const int unit = blockIdx.x / CG;
  const int units = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    for (int pi = 0; pi < g.nprob; ++pi) {
      const Prob& P = g.p[pi];
      tma_prefetch_desc(&tm.m[MAPS_PER_PROB * pi]);
      tma_prefetch_desc(&tm.m[MAPS_PER_PROB * pi + 1]);
      if (P.epi == EPI_DW || P.a.tma_out) tma_prefetch_desc(&tm.m[MAPS_PER_PROB * pi + 2]);
      if (P.a_split != NO_SPLIT) tma_prefetch_desc(&tm.m[MAPS_PER_PROB * pi + 3]);
      if (P.c_split != NO_SPLIT) tma_prefetch_desc(&tm.m[MAPS_PER_PROB * pi + 4]);
    }
#pragma unroll
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4 * CG);  // one arrive per epilogue warp of every CTA of the pair
    }
    for (int i = 0; i < 4; ++i) mbar_init(&sbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2)
      tmem_alloc_pair<TMEM_COLS>(tmem_slot);
    else
      tmem_alloc<TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync();
    __syncthreads();  // also a CTA barrier, so race checkers that do not model barrier.cluster see
                      // the TMEM address written by tcgen05.alloc ordered before the reads below
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: let the next launch's CTAs start their prologue as soon as SMs free up, and wait for the
  // previous grid (whose outputs we read, and whose inputs we may overwrite) before any global access.
  griddep_launch_dependents();
  if (!g.early || warp >= 2) griddep_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs of a pair load their own halves) =====
      const uint64_t pol = policy_evict_normal();
      uint32_t stage = 0, phase = 0;
      unsigned long long u_ew = 0;
      const bool tu = (g.dbg & 4) && unit < TRACE_UNITS && rank == 0;
      // in-kernel combine: the stash flagged a possible in-place rescale -> wait before any load;
      // else only the dW tiles (B = X'^T, written by the combine) wait
      bool cj_wait = g.cj_on != 0;
      const bool cj_all = cj_wait && ld_relaxed_u32(g.cj.fb_flag) != 0;
      TileIter it(g, unit, units);
      for (Item item = it.next_item(); item.tile >= 0; item = it.next_item()) {
        const int tile = item.tile;
        const int pi = prob_of(g, tile);
        const Prob& P = g.p[pi];
        if (cj_wait && (cj_all || P.epi == EPI_DW)) {
          spin_until_geq(g.cj.counter, gridDim.x);
          fence_proxy_async_global();  // the combine's generic stores before these TMA reads
          cj_wait = false;
        }
        const CUtensorMap* tA = &tm.m[MAPS_PER_PROB * pi];
        const CUtensorMap* tB = &tm.m[MAPS_PER_PROB * pi + 1];
        const CUtensorMap* tA2 = &tm.m[MAPS_PER_PROB * pi + 3];
        int m_blk, n_blk;
        tile_coords(tile - P.tile_begin, P.a, m_blk, n_blk);
        const int a_row = m_blk * C::TILE_M + (int)rank * BM;
        const int b_row = n_blk * BN + (int)rank * C::B_ROWS;
        const int kb_beg = item.kb0, kb_end = g.il ? item.kb1 : (P.a.K + BK - 1) / BK;
        const bool a_mn = P.a_mn, b_mn = P.b_mn;
        if (g.dbg & 8) {  // experiment: pull the next tile's MN-major A operand (all of K) into L2
          const int nt = it.peek();
          if (nt >= 0) {
            const int npi = prob_of(g, nt);
            const Prob& Q = g.p[npi];
            if (Q.a_mn && !Q.a3d) {
              int nm, nn;
              tile_coords(nt - Q.tile_begin, Q.a, nm, nn);
              const int nrow = nm * C::TILE_M + (int)rank * BM;
              const int nkb = (Q.a.K + BK - 1) / BK;
              for (int kb = 0; kb < nkb; ++kb) {
                const CUtensorMap* m = &tm.m[MAPS_PER_PROB * npi];
                int k = kb * BK;
                if (k >= Q.a_split) { m = &tm.m[MAPS_PER_PROB * npi + 3]; k -= Q.a_split; }
                for (int j = 0; j < BM / 64; ++j) tma_prefetch_l2_2d(m, nrow + j * 64, k);
              }
            }
          }
        }
        for (int kb = kb_beg; kb < kb_end; ++kb) {
          unsigned long long c0 = tu ? clk() : 0;
          mbar_wait(&empty[stage], phase ^ 1);
          if (tu) u_ew += clk() - c0;
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          // A's outer (row) coordinate: M for K-major A, K for MN-major A; rows >= a_split come
          // from the second segment's map.
          const CUtensorMap* tAk = tA;
          int a_r = a_row, a_k = kb * BK;
          if ((g.dbg & 2048) && a_mn) a_k = (kb & 1) * BK;  // timing experiment only: L2-resident MN-major A (wrong)
          if (!a_mn) {
            if (a_r >= P.a_split) { tAk = tA2; a_r -= P.a_split; }
          } else if (a_k >= P.a_split) {
            tAk = tA2;
            a_k -= P.a_split;
          }
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            if (!a_mn) {
              tma_load_2d(tAk, &full[stage], a_dst, a_k, a_r, pol);
            } else if (P.a3d) {
              tma_load_3d(tAk, &full[stage], a_dst, 0, a_k, a_r / 64, pol);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_2d(tAk, &full[stage], a_dst + j * 8192, a_r + j * 64, a_k, pol);
            }
            if (!b_mn) {
              tma_load_2d(tB, &full[stage], b_dst, kb * BK, b_row, pol);
            } else if (P.b3d) {
              tma_load_3d(tB, &full[stage], b_dst, 0, kb * BK, b_row / 64, pol);
            } else {
#pragma unroll
              for (int j = 0; j < C::B_ROWS / 64; ++j)
                tma_load_2d(tB, &full[stage], b_dst + j * 8192, b_row + j * 64, kb * BK, pol);
            }
          } else {
            // Both CTAs' bytes complete on the leader's full barrier; only the leader arrives.
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES * 2);
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            if (!a_mn) {
              tma_load_2d_pair(tAk, fb, a_dst, a_k, a_r, pol);
            } else if (P.a3d) {
              tma_load_3d_pair(tAk, fb, a_dst, 0, a_k, a_r / 64, pol);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(tAk, fb, a_dst + j * 8192, a_r + j * 64, a_k, pol);
            }
            if (!b_mn) {
              tma_load_2d_pair(tB, fb, b_dst, kb * BK, b_row, pol);
            } else if (P.b3d) {
              tma_load_3d_pair(tB, fb, b_dst, 0, kb * BK, b_row / 64, pol);
            } else {
#pragma unroll
              for (int j = 0; j < C::B_ROWS / 64; ++j)
                tma_load_2d_pair(tB, fb, b_dst + j * 8192, b_row + j * 64, kb * BK, pol);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (tu) g_trace[TRACE_TILES * 8 + unit * 8 + 5] = u_ew;
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== tcgen05.mma issuer (pair leader only) =====
      uint32_t stage = 0, phase = 0, local = 0, ntiles = 0;
      uint32_t uses0 = 0, uses1 = 0;  // completed accumulations per TMEM slot (scalars: no local memory)
      unsigned long long u_fw = 0, u_tw = 0, u_kb = 0, u_first = 0, u_gt0 = 0;
      TileIter it(g, unit, units);
      for (Item item = it.next_item(); item.tile >= 0; item = it.next_item(), ++local) {
        const int tile = item.tile;
        const Prob& P = g.p[prob_of(g, tile)];
        const bool a_mn = P.a_mn, b_mn = P.b_mn;
        const uint32_t idesc = make_idesc_bf16(C::TILE_M, BN, a_mn, b_mn);
        const int kb_beg = item.kb0, kb_end = g.il ? item.kb1 : (P.a.K + BK - 1) / BK;
        const uint32_t acc = item.slot >= 0 ? (uint32_t)item.slot : (ntiles & 1);
        if (item.first) ++ntiles;
        const uint32_t acc_phase = (acc ? uses1 : uses0) & 1;
        const bool tr = (g.dbg & 4) && blockIdx.x == 0 && local < TRACE_TILES;
        const bool tu = (g.dbg & 4) && unit < TRACE_UNITS;
        unsigned long long c0 = 0;
        if (tu) {
          c0 = clk();
          if (local == 0) {
            u_first = c0;
            u_gt0 = gtimer();
          }
        }
        if (tr) g_trace[local * 8 + 0] = clk();
        if (item.first) {  // the accumulator must be free (its previous tile's epilogue released it)
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
        }
        if (tu) u_tw += clk() - c0;
        if (tr) g_trace[local * 8 + 1] = clk();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb_beg; kb < kb_end; ++kb) {
          if (tu) c0 = clk();
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (tu) {
            u_fw += clk() - c0;
            ++u_kb;
          }
          const uint32_t a_base = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = a_mn ? make_sdesc(a_base + k * 2048, 8192, 1024) : make_sdesc(a_base + k * 32, 16, 1024);
            const uint64_t bd = b_mn ? make_sdesc(b_base + k * 2048, 8192, 1024) : make_sdesc(b_base + k * 32, 16, 1024);
            const bool accum = !(item.first && kb == kb_beg && k == 0);
            if constexpr (CG == 2)
              mma_bf16_pair(d_tmem, ad, bd, idesc, accum);
            else
              mma_bf16(d_tmem, ad, bd, idesc, accum);
          }
          // frees the smem slot (in both CTAs) once these MMAs have read it
          if constexpr (CG == 2)
            mma_commit_pair(&empty[stage], 0x3);
          else
            mma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        // accumulator ready for the epilogue warps (of both CTAs) once the tile's last segment is in
        if (item.last) {
          if constexpr (CG == 2)
            mma_commit_pair(&tfull[acc], 0x3);
          else
            mma_commit(&tfull[acc]);
          if (acc) ++uses1; else ++uses0;
        }
        if (tr) g_trace[local * 8 + 2] = clk();
      }
      if ((g.dbg & 4) && unit < TRACE_UNITS) {
        unsigned long long* u = g_trace + TRACE_TILES * 8 + unit * 8;
        u[0] = u_fw;
        u[1] = u_tw;
        u[2] = u_first;
        u[3] = clk();
        u[4] = u_kb;
        u[6] = local;
        u[7] = gtimer() - u_gt0;
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: thread = TMEM lane = output row =====
    const uint32_t ew = warp - 4;
    if (g.cj_on) {  // the chunk's combine, rows spread over every CTA of the launch
      const int tid = (int)(ew * 32 + lane);
      combine_rows_dev(g.cj, (int)blockIdx.x, (int)gridDim.x, tid, 1, reinterpret_cast<float*>(stg));
      __threadfence();
      named_bar_sync(1, 128);
      if (tid == 0) {
        atomicAdd(g.cj.counter, 1u);
        spin_until_geq(g.cj.counter, gridDim.x);  // RowStat / row factors of every row
      }
      named_bar_sync(1, 128);
    }
    uint32_t local = 0;
    uint32_t sphase = 0;  // parity bits of the two staging barriers
    uint32_t sq = 0;      // staging-buffer sequence of the chunk-pipelined dW epilogue
    uint32_t ntiles = 0, uses0 = 0, uses1 = 0;
    TileIter it(g, unit, units);
    for (Item item = it.next_item(); item.tile >= 0; item = it.next_item()) {
      const int tile = item.tile;
      const uint32_t acc = item.slot >= 0 ? (uint32_t)item.slot : (ntiles & 1);
      if (item.first) ++ntiles;
      if (!item.last) continue;  // an interior K segment: the accumulation goes on
      const uint32_t acc_phase = (acc ? uses1++ : uses0++) & 1;
      const int pi = prob_of(g, tile);
      const Prob& P = g.p[pi];
      int m_blk, n_blk;
      tile_coords(tile - P.tile_begin, P.a, m_blk, n_blk);
      const bool tr = (g.dbg & 4) && blockIdx.x == 0 && local < TRACE_TILES && ew == 0 && lane == 0;
      if (tr) {
        g_trace[local * 8 + 3] = clk();
        g_trace[local * 8 + 7] = pi;
      }
      auto wait_acc = [&]() {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (tr) g_trace[local * 8 + 4] = clk();
      };
      const uint32_t taddr = tmem_base + ((ew * 32) << 16) + acc * BN;
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (tr) g_trace[local * 8 + 5] = clk();
        if (lane == 0) {
          if constexpr (CG == 2)
            mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          else
            mbar_arrive(&tempty[acc]);
        }
      };
      if (P.epi == EPI_DW) {
        // Warm L2 with the old dW rows of this unit's next tile while this one is processed.
        const int nt = it.peek();
        if (ew == 0 && lane == 0 && nt >= 0 && !(g.dbg & 1)) {
          const int npi = prob_of(g, nt);
          const Prob& Q = g.p[npi];
          if (Q.epi == EPI_DW && Q.a.mode == 1) {
            int qm, qn;
            tile_coords(nt - Q.tile_begin, Q.a, qm, qn);
            for (int k = 0; k < BN / 64 && qn * BN + k * 64 < Q.a.N; ++k)
              tma_prefetch_l2_2d(&tm.m[MAPS_PER_PROB * npi + 2], qn * BN + k * 64, qm * C::TILE_M + (int)rank * BM);
          }
        }
        epilogue_dw_tma<NB>(P.a, &tm.m[MAPS_PER_PROB * pi + 2], taddr, m_blk * C::TILE_M + (int)rank * BM, n_blk,
                        ew * 32 + lane, stg, sbar, sphase, sq, ew == 0 && lane == 0, wait_acc, release, g.dbg);
      } else if (P.epi == EPI_STASH && P.a.tma_out) {  // a stash tensor map is provided
        const int row0 = m_blk * C::TILE_M + (int)rank * BM;  // output rows >= c_split go to map C2
        const bool seg2 = row0 >= P.c_split;
        epilogue_stash_tma<NB>(P.a, &tm.m[MAPS_PER_PROB * pi + (seg2 ? 4 : 2)], taddr, row0, n_blk, ew * 32 + lane,
                           stg, ew == 0 && lane == 0, wait_acc, release, sq, seg2 ? P.c_split : 0);
      } else {
        wait_acc();
        epilogue_dispatch(P.epi, P.a, taddr, m_blk * C::TILE_M + (int)rank * BM, n_blk, ew * 32 + lane);
        release();
      }
      if (tr) g_trace[local * 8 + 6] = clk();
      ++local;
    }
  }
  if (warp == 4 && lane == 0) bulk_wait<0>();  // epilogue TMA stores complete before exit
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc_pair<TMEM_COLS>(tmem_base);
    else
      tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

}  // namespace slf
