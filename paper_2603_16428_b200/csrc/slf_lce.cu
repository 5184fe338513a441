// slf_lce.cu — host side of libslf_lce.so: argument checks, the schedule planner, TMA descriptor
// construction and the launch sequence of the fused LCE hot path (include/slf_lce.h,
// DESIGN.md §Boundary, §Schedules).  Device code lives in gemm.cuh and aux_kernels.cuh.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/slf_lce.h"
#include "aux_kernels.cuh"
#include "gemm.cuh"
#include "rmsnorm.cuh"
#include "s_kernels.cuh"
#include "comm.cuh"

using namespace slf;

namespace {

thread_local std::string g_err;

slf_status fail(slf_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define SLF_CUDA(x)                                                                                        \
  do {                                                                                                     \
    cudaError_t e_ = (x);                                                                                  \
    if (e_ != cudaSuccess) return fail(SLF_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define SLF_TRY(x)                   \
  do {                               \
    slf_status s_ = (x);             \
    if (s_ != SLF_OK) return s_;     \
  } while (0)

constexpr int kMaxDev = 64;

// ---- instrumentation (slf_profile_begin/end) ---------------------------------------------------
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
  double flops, bytes;
};
struct ProfState {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
};
thread_local ProfState g_prof;

cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// RAII bracket around one launch; no-op unless profiling is on.
struct ProfScope {
  int idx = -1;
  cudaStream_t s;
  ProfScope(int kind, cudaStream_t s_, double flops, double bytes) : s(s_) {
    if (!g_prof.on) return;
    ProfRec r{kind, prof_event(), prof_event(), flops, bytes};
    cudaEventRecord(r.a, s);
    g_prof.recs.push_back(r);
    idx = (int)g_prof.recs.size() - 1;
  }
  ~ProfScope() {
    if (idx >= 0) cudaEventRecord(g_prof.recs[idx].b, s);
  }
};

// Pinned host staging ring for the per-call tile tables: an H2D cudaMemcpyAsync from pageable
// memory may synchronise with the stream (the GPU would idle while the host enqueues the next
// call); from pinned memory it is asynchronous.  A slot is reused only after the event recorded
// behind its copy has completed (in practice never waited on: 8 calls in flight).
constexpr int RING_SLOTS = 8;
struct PinnedRing {
  uint8_t* buf = nullptr;
  cudaEvent_t ev[RING_SLOTS] = {};
  bool used[RING_SLOTS] = {};
  int next = 0;
};

struct DevInfo {
  int sms = 0;
  int major = 0;
  int minor = 0;
  bool gemm_attr_set[64] = {};
  PinnedRing ring;
  // slf_lce_fwd_bwd_host: copy stream and per-chunk events (created on first use)
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> copy_events;
  // per staging buffer (hidden_dev): recorded at the end of the last call that read it, so the next
  // call's copy into it waits only for that call, not for everything on the stream (double-buffered
  // staging lets step k+1's input copy run under step k)
  std::map<const void*, cudaEvent_t> staging_free;
};

std::mutex g_mu;
DevInfo g_dev[kMaxDev];

slf_status device_info(DevInfo** out) {
  int dev = 0;
  SLF_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) return fail(SLF_ERR_UNSUPPORTED, "device ordinal %d out of range", dev);
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo& d = g_dev[dev];
  if (d.sms == 0) {
    SLF_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    SLF_CUDA(cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev));
    SLF_CUDA(cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev));
  }
  if (d.major != 10 || d.minor != 0)
    return fail(SLF_ERR_UNSUPPORTED, "libslf_lce is built for sm_100a; device is sm_%d%d", d.major, d.minor);
  *out = &d;
  return SLF_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map, dims {inner (contiguous), outer}, 128-byte swizzle, zero fill out of bounds.
slf_status make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                     uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return fail(SLF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SLF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu stride %llu box %u x %u", (int)r,
                (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_stride_bytes, box_inner,
                box_outer);
  return SLF_OK;
}
// Operand views.  K-major: stored [rows][K] -> box {64, rows_per_tile}.  MN-major: stored [K][MN]
// -> box {64, 64}, several boxes per stage.
slf_status tmap_kmajor(CUtensorMap* m, const void* base, int64_t K, int64_t rows, int64_t ld, uint32_t box_rows) {
  return make_tmap(m, base, (uint64_t)K, (uint64_t)rows, (uint64_t)ld * 2, 64, box_rows);
}
// MN-major operands with MN % 64 == 0 use a 3-D map {64 MN, K, MN/64} (strides ld*2 and 128 bytes)
// and one box {64, 64, atoms} per stage: the same bytes and shared-memory layout ([atom][64 K][64
// MN], atoms 8 KB apart) as `atoms` 2-D boxes, in one TMA instruction.  Two MN-major operands in
// 2-D boxes issue four TMA loads per stage and ran ~10 % below one K-major operand (debug GEMM,
// 587 vs 533-543 cycles per K-block); SLF_MN3D=0 keeps the 2-D boxes.
slf_status make_tmap_mn3d(CUtensorMap* m, const void* base, uint64_t MN, uint64_t K, uint64_t ld_bytes, uint32_t atoms) {
  auto fn = encode_fn();
  if (!fn) return fail(SLF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, K, (MN + 63) / 64};  // MN % 64 != 0: the last atom reads past MN (see s_build_bwd)
  cuuint64_t strides[2] = {ld_bytes, 128};
  cuuint32_t box[3] = {64, 64, atoms};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SLF_ERR_CUDA, "cuTensorMapEncodeTiled (3-D MN-major) failed (%d): MN %llu K %llu ld %llu", (int)r,
                (unsigned long long)MN, (unsigned long long)K, (unsigned long long)ld_bytes);
  return SLF_OK;
}

// Whether 3-D MN-major maps are used (decided once: the environment, then a trial encoding).
bool mn3d_enabled() {
  static const bool on = [] {
    const char* e = getenv("SLF_MN3D");
    if (e && atoi(e) == 0) return false;
    static uint16_t probe[64 * 64 * 2];
    CUtensorMap m;
    const std::string keep = g_err;
    const bool ok = make_tmap_mn3d(&m, probe, 128, 64, 128 * 2, 2) == SLF_OK;
    g_err = keep;
    return ok;
  }();
  return on;
}

bool mn3d_for(int64_t MN) { return MN % 64 == 0 && mn3d_enabled(); }

// `atoms`: 64-wide MN atoms per stage of this operand (A: BM/64; B: (BN/cta_group)/64).
slf_status tmap_mnmajor(CUtensorMap* m, const void* base, int64_t MN, int64_t K, int64_t ld, uint32_t atoms = 2) {
  if (mn3d_for(MN)) return make_tmap_mn3d(m, base, (uint64_t)MN, (uint64_t)K, (uint64_t)ld * 2, atoms);
  return make_tmap(m, base, (uint64_t)MN, (uint64_t)K, (uint64_t)ld * 2, 64, 64);
}

// CTA-group selection: 2 (CTA pairs, 256 x 256 tiles; default) or 1 (128 x 256), env SLF_CTA_GROUP.
int cta_group() {
  static int cg = [] {
    const char* e = getenv("SLF_CTA_GROUP");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return cg;
}
uint32_t b_box_rows() { return (uint32_t)(BN / cta_group()); }

// One GEMM problem of a launch: operand tensor maps, extents and epilogue arguments.
struct ProbSpec {
  CUtensorMap ta, tb, tc;  // tc: TMA-staged output map (EPI_DW, EPI_STASH)
  CUtensorMap ta2, tc2;    // second row segment of A / of the output (see Prob::a_split / c_split)
  GemmArgs a{};
  int epi = EPI_F32;
  bool a_mn = false, b_mn = false;
  int a_split = NO_SPLIT, c_split = NO_SPLIT;
  bool a3d_force = false;  // ta is a 3-D MN-major map although M % 64 != 0 (over-read is harmless)
  bool ro_operands = false;  // A and B are call inputs no kernel writes (GroupArgs::early)
};

int prof_kind_of(int epi) {
  switch (epi) {
    case EPI_STATS:
    case EPI_STASH: return SLF_PROF_GEMM_STATS;
    case EPI_GRAD: return SLF_PROF_GEMM_GRAD;
    case EPI_DW: return SLF_PROF_GEMM_DW;
    case EPI_DX:
    case EPI_DXS: return SLF_PROF_GEMM_DX;
    default: return SLF_PROF_GEMM_DEBUG;
  }
}

void finish_geometry(GemmArgs& a, int cg) {
  const int tile_m = BM * cg;
  a.tiles_m = (a.M + tile_m - 1) / tile_m;
  a.tiles_n = (a.N + BN - 1) / BN;
  a.num_tiles = a.tiles_m * a.tiles_n;
  static const int gm = getenv("SLF_GROUP_M") ? atoi(getenv("SLF_GROUP_M")) : 16 / cg;  // raster experiments
  a.group_m = std::max(1, std::min(a.tiles_m, gm));
}

// Interleaved schedule of a schedule-S group (the chunk's dX GEMM, K = V, and dW GEMM, K = rows),
// DESIGN.md §6 (experiment, SLF_INTERLEAVE=1): each of the T0 <= units dX tiles belongs to one unit and is split into K segments of
// L K-blocks; after segment s of every dX tile, the dW tiles whose vocabulary rows are that segment's
// K range (the same stash columns) go to the least-loaded units.  The stash slab and the W rows a
// segment streams are then read again by those dW tiles while they are still in L2, instead of
// long after (round 1: all dX tiles first, dW tiles afterwards); a dX accumulation stays open in TMEM
// slot 0 across its segments while its unit's dW tiles use slot 1 (their epilogues overlap the next
// segment).  Returns (tile, seg) int pairs per unit and a NEGATIVE stride (the kernel's il mode), or
// an empty table when the group does not have that shape.
int host_m_blk(const GemmArgs& a, int tile) {
  const int per_group = a.group_m * a.tiles_n;
  const int gi = tile / per_group;
  const int first_m = gi * a.group_m;
  const int gm = std::min(a.group_m, a.tiles_m - first_m);
  return first_m + (tile - gi * per_group) % gm;
}

std::vector<int> interleave_table(const ProbSpec* ps, int n, int units, int* stride) {
  static const int seg_env = getenv("SLF_IL_SEG") ? atoi(getenv("SLF_IL_SEG")) : 16;
  // Off by default (SLF_INTERLEAVE=1 selects it): it cuts the group's DRAM reads by 10 % but issues
  // 5–10 % fewer MMAs per clock (measured), so the step is not faster.
  static const bool off = !(getenv("SLF_INTERLEAVE") && atoi(getenv("SLF_INTERLEAVE")) == 1);
  if (off || n != 2 || ps[0].epi != EPI_DXS || ps[1].epi != EPI_DW) return {};
  const GemmArgs &ax = ps[0].a, &aw = ps[1].a;
  const int T0 = ax.num_tiles, T1 = aw.num_tiles;
  const int KB0 = (ax.K + BK - 1) / BK, KB1 = (aw.K + BK - 1) / BK;
  const int mkb = BM * cta_group() / BK;  // dX K-blocks per dW row tile (the same vocabulary rows)
  const int L = std::max(mkb, seg_env / mkb * mkb);
  if (T0 < 1 || T0 > units || T1 < 1 || KB0 >= 4096 || KB1 >= 4096 || aw.M * 1LL != ax.K * 1LL) return {};
  const int S = (KB0 + L - 1) / L;
  std::vector<std::vector<int>> bucket(S);
  for (int t = 0; t < T1; ++t) bucket[std::min(S - 1, host_m_blk(aw, t) * mkb / L)].push_back(t);
  std::vector<std::vector<int>> items(units);
  std::vector<long long> load(units, 0);
  std::vector<int> alt(units, 0);
  static const int ovh = getenv("SLF_LPT_OVH") ? atoi(getenv("SLF_LPT_OVH")) : 4;
  auto seg = [](int kb0, int kb1, int first, int last, int slot) {
    return kb0 | (kb1 << 12) | (first << 24) | (last << 25) | (slot << 26);
  };
  for (int s = 0; s < S; ++s) {
    for (int u = 0; u < T0; ++u) {
      const int kb0 = s * L, kb1 = std::min(KB0, kb0 + L);
      items[u].push_back(u);
      items[u].push_back(seg(kb0, kb1, s == 0, kb1 == KB0, 0));
      load[u] += kb1 - kb0;
    }
    for (int t : bucket[s]) {
      int best = 0;
      for (int u = 1; u < units; ++u)
        if (load[u] < load[best]) best = u;
      const int slot = best < T0 ? 1 : (alt[best]++ & 1);
      items[best].push_back(T0 + t);
      items[best].push_back(seg(0, KB1, 1, 1, slot));
      load[best] += KB1 + ovh;
    }
  }
  size_t mx = 2;
  for (auto& l : items) mx = std::max(mx, l.size() + 2);
  std::vector<int> tab((size_t)units * mx, -1);
  for (int u = 0; u < units; ++u)
    for (size_t i = 0; i < items[u].size(); ++i) tab[(size_t)u * mx + i] = items[u][i];
  *stride = -(int)mx;
  return tab;
}

// Longest-processing-time-first assignment of the tiles of a group to `units` persistent units:
// tiles sorted by K-blocks (descending, stable by id), each given to the least-loaded unit.
// Returns a [units][stride] table of tile ids, -1 padded.  (With SLF_INTERLEAVE=1 a schedule-S
// dX + dW group gets the interleaved table above instead.)
std::vector<int> lpt_table(const ProbSpec* ps, int n, int units, int* stride) {
  {
    std::vector<int> il = interleave_table(ps, n, units, stride);
    if (!il.empty()) return il;
  }
  std::vector<std::pair<int, int>> tiles;  // (kblocks, id)
  int id = 0;
  for (int p = 0; p < n; ++p) {
    const int kb = (ps[p].a.K + BK - 1) / BK;
    // Cost in K-blocks plus a per-tile epilogue/pipeline overhead; a dW read-modify-write tile
    // pays extra for streaming the old partial (SLF_LPT_OVH / SLF_LPT_RMW tune the model).
    // 3: per-unit MMA spans of a Llama-8B group within 2 % (4: the dX units ended 3.5 % after the
    // dW-only units; group 29.6 vs 29.9 ms per step, profiles/r02/lpt_ovh.md)
    static const int ovh = getenv("SLF_LPT_OVH") ? atoi(getenv("SLF_LPT_OVH")) : 3;
    static const int rmw = getenv("SLF_LPT_RMW") ? atoi(getenv("SLF_LPT_RMW")) : 0;
    const int cost = kb + ovh + ((ps[p].epi == EPI_DW && ps[p].a.mode == 1) ? rmw : 0);
    for (int t = 0; t < ps[p].a.num_tiles; ++t) tiles.push_back({cost, id++});
  }
  std::stable_sort(tiles.begin(), tiles.end(), [](auto& x, auto& y) { return x.first > y.first; });
  std::vector<std::vector<int>> lists(units);
  std::vector<long long> load(units, 0);
  for (auto& t : tiles) {
    int best = 0;
    for (int u = 1; u < units; ++u)
      if (load[u] < load[best]) best = u;
    lists[best].push_back(t.second);
    load[best] += t.first;
  }
  // Order within a unit (experiment knob SLF_LPT_ORDER=mid): move the unit's longest tile (assigned
  // first) to the middle of its list so long-K and short-K tiles overlap in time across units.
  static const bool mid = getenv("SLF_LPT_ORDER") && std::string(getenv("SLF_LPT_ORDER")) == "mid";
  if (mid)
    for (auto& l : lists)
      if (l.size() > 2) std::rotate(l.begin(), l.begin() + 1, l.begin() + 1 + l.size() / 2);
  size_t mx = 1;
  for (auto& l : lists) mx = std::max(mx, l.size() + 1);
  *stride = (int)mx;
  std::vector<int> tab((size_t)units * mx, -1);
  for (int u = 0; u < units; ++u)
    for (size_t i = 0; i < lists[u].size(); ++i) tab[(size_t)u * mx + i] = lists[u][i];
  return tab;
}

// SMs the GEMM launches may use.  The vocab-sharded call can leave some to the communicator's
// kernels: the persistent GEMM CTAs (1 per SM, ~226 KB shared memory, 237 registers per thread)
// leave no room for an NCCL block, so without reserved SMs the dX all-reduce of chunk c can only
// run between launches instead of under the next chunk's stash GEMM.  Thread-local:
// set by phase_sharded for the duration of one call.
thread_local int tl_reserved_sms = 0;
int usable_sms(const DevInfo* dev) {
  const int r = std::min(std::max(tl_reserved_sms, 0), dev->sms - 2);
  return (dev->sms - r) & ~1;  // whole CTA pairs
}
struct ReserveSms {
  int prev;
  explicit ReserveSms(int n) : prev(tl_reserved_sms) { tl_reserved_sms = n; }
  ~ReserveSms() { tl_reserved_sms = prev; }
};

template <int CG, int NB>
slf_status launch_group_cfg(DevInfo* dev, ProbSpec* ps, int n, cudaStream_t s, const int* sched, int sched_stride,
                            int prof_kind, const CombineJob* cj = nullptr) {
  using C = Cfg<CG, NB>;
  auto kfn = lce_group_kernel<CG, NB>;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!dev->gemm_attr_set[CG * 8 + NB]) {
      SLF_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
      dev->gemm_attr_set[CG * 8 + NB] = true;
    }
  }
  TMaps tm;
  GroupArgs g{};
  int total = 0;
  double flops = 0;
  int np = 0;
  for (int p = 0; p < n; ++p) {
    GemmArgs a = ps[p].a;
    if (a.M <= 0 || a.N <= 0 || a.K <= 0) continue;
    finish_geometry(a, CG);
    tm.m[MAPS_PER_PROB * np] = ps[p].ta;
    tm.m[MAPS_PER_PROB * np + 1] = ps[p].tb;
    tm.m[MAPS_PER_PROB * np + 2] = ps[p].tc;
    tm.m[MAPS_PER_PROB * np + 3] = ps[p].ta2;
    tm.m[MAPS_PER_PROB * np + 4] = ps[p].tc2;
    g.p[np] = Prob{a, ps[p].epi, ps[p].a_mn ? 1 : 0, ps[p].b_mn ? 1 : 0, total, ps[p].a_split, ps[p].c_split,
                   (ps[p].a_mn && (ps[p].a3d_force || mn3d_for(a.M))) ? 1 : 0,
                   (ps[p].b_mn && mn3d_for(a.N)) ? 1 : 0};
    total += a.num_tiles;
    flops += 2.0 * a.M * a.N * (double)a.K;
    ++np;
  }
  if (np == 0) return SLF_OK;
  g.nprob = np;
  g.num_tiles = total;
  g.sched = sched;
  g.sched_stride = sched_stride < 0 ? -sched_stride : sched_stride;  // negative: interleaved (seg) table
  g.il = sched && sched_stride < 0 ? 1 : 0;
  if (cj) {  // every CTA of the launch arrives once; the grid is one persistent CTA per usable SM
    g.cj_on = 1;
    g.cj = *cj;
  }
  static const bool early_off = getenv("SLF_EARLY_MAINLOOP") && atoi(getenv("SLF_EARLY_MAINLOOP")) == 0;
  static const int dbg = getenv("SLF_DEBUG_EPI") ? atoi(getenv("SLF_DEBUG_EPI")) : 0;  // timing experiments only
  g.dbg = dbg & ~4;
  {  // SLF_DEBUG_TRACE=k: record the per-tile trace of the k-th group launch of this process
    static const int trace_at = getenv("SLF_DEBUG_TRACE") ? atoi(getenv("SLF_DEBUG_TRACE")) : -1;
    static int launch_no = 0;
    if (launch_no++ == trace_at) g.dbg |= 4;
  }
  const int units = sched ? usable_sms(dev) / CG : std::min(total, usable_sms(dev) / CG);
  // Early mainloop (stash GEMM of chunk >= 1, s_chunk_stats): it can only launch once the previous
  // group launch is fully resident, which cannot happen while the call's first stash GEMM still
  // waits for the kernels before the call as long as this grid plus a full group grid exceed the
  // SMs (not so with a tiny grid next to many SMs left to a communicator).
  g.early = (!early_off && np == 1 && !sched && ps[0].ro_operands && units * CG + usable_sms(dev) > dev->sms) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * CG));
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // Programmatic dependent launch: this grid's CTAs may start (prologue: barrier init, TMEM
  // alloc, descriptor prefetch) while the previous kernel drains; griddepcontrol.wait in the
  // kernel holds every global-memory access until the previous grid has completed.
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  ProfScope pscope(prof_kind >= 0 ? prof_kind : prof_kind_of(g.p[0].epi), s, flops, 0.0);
  SLF_CUDA(cudaLaunchKernelEx(&cfg, kfn, tm, g));
  return SLF_OK;
}

// How a dW partial is accumulated into the previous one.  2 (default): the epilogue rounds its
// fp32 partial to bf16 and a TMA reduce-add store has the L2 add it to dW (cp.reduce.async.bulk
// .tensor .add, bf16) — nothing is loaded through the SM, so the short-K dW tiles stay fed and
// the launch keeps the 6-stage ring.  1: the epilogue loads the old bf16 tile by TMA, adds in fp32
// and stores (one rounding instead of two; measured max error identical, but
// ~2.5 ms per Llama-8B step slower).  SLF_DW_ACC=1 selects it.
int dw_acc_mode() {
  static const int m = getenv("SLF_DW_ACC") ? atoi(getenv("SLF_DW_ACC")) : 2;
  return m == 1 ? 1 : 2;
}

// Launch configuration: a launch with a dW read-modify-write problem keeps four epilogue staging
// buffers (5-stage ring); every other launch takes the 6-stage ring (SLF_STAGING=2|4 forces one,
// timing experiments only).
slf_status launch_group(DevInfo* dev, ProbSpec* ps, int n, cudaStream_t s, const int* sched = nullptr,
                        int sched_stride = 0, int prof_kind = -1, const CombineJob* cj = nullptr) {
  bool dw = false;
  for (int p = 0; p < n; ++p) dw = dw || (ps[p].epi == EPI_DW && ps[p].a.mode == 1);
  static const int force = getenv("SLF_STAGING") ? atoi(getenv("SLF_STAGING")) : 0;
  const bool four = force ? force == 4 : dw;
  if (cta_group() == 2)
    return four ? launch_group_cfg<2, 4>(dev, ps, n, s, sched, sched_stride, prof_kind, cj)
                : launch_group_cfg<2, 2>(dev, ps, n, s, sched, sched_stride, prof_kind, cj);
  return four ? launch_group_cfg<1, 4>(dev, ps, n, s, sched, sched_stride, prof_kind, cj)
              : launch_group_cfg<1, 2>(dev, ps, n, s, sched, sched_stride, prof_kind, cj);
}

template <int EPI, bool A_MN, bool B_MN>
slf_status launch_gemm(DevInfo* dev, const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs a, cudaStream_t s) {
  ProbSpec p;
  p.ta = ta;
  p.tb = tb;
  p.a = a;
  p.epi = EPI;
  p.a_mn = A_MN;
  p.b_mn = B_MN;
  return launch_group(dev, &p, 1, s);
}

// ---- planner (schedule R) ----------------------------------------------------------------------
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Plan {
  int sched = SLF_SCHED_R;
  // schedule R: row block R x vocab chunk Cv
  int64_t R = 0, Cv = 0, nR = 0, nC = 0;
  // schedule S: row chunk C (whole vocabulary stashed per chunk)
  int64_t C = 0, nCh = 0, ld_stash = 0;
  size_t sched_bytes = 0;
  size_t off_sched = 0, off_rowstat = 0, off_shard = 0, off_zt = 0, off_union = 0, off_dxacc = 0;
  size_t off_loss = 0, off_cnt = 0, off_off = 0, off_hits = 0, off_idx = 0, off_part = 0, off_stash = 0;
  size_t off_mref = 0, off_fac = 0;  // schedule S: per-row stash reference and row factor [N] fp32
  size_t fwd_bytes = 0, bwd_bytes = 0, total = 0;
};

// LPT tile-table arena: up to 8 tables of a group launch, each <= 2 x (tiles + units) ints, with
// tiles <= (ceil(N/128) + ceil(V/128)) * ceil(H/256); clamped to [64 KB, 1 MB] (a call needing more
// uploads one table per launch instead, phase_s).
constexpr size_t SCHED_ARENA_MAX = 1024 * 1024;
size_t sched_arena_bytes(int64_t N, int64_t H, int64_t V) {
  const double tiles = (double)((N + 127) / 128 + (V + 127) / 128) * (double)((H + 255) / 256);
  const double b = 8.0 * (2.0 * tiles + 2.0 * 148) * 4.0;
  return align_up((size_t)std::min<double>((double)SCHED_ARENA_MAX, std::max<double>(64.0 * 1024, b)), 1024);
}

size_t default_budget(int64_t N, int64_t V) {
  const size_t five = (size_t)(0.05 * (double)N * (double)V * 2.0);
  return std::max(five, (size_t)16 << 20);
}

bool plan_r(int64_t N, int64_t H, int64_t V, size_t budget, Plan* out) {
  if (N < 1 || H < 8 || V < 1) return false;
  if (budget == 0) budget = default_budget(N, V);
  Plan p;
  p.sched = SLF_SCHED_R;
  p.off_sched = WS_HEADER_BYTES;
  p.sched_bytes = sched_arena_bytes(N, H, V);
  p.off_rowstat = p.off_sched + p.sched_bytes;
  p.off_shard = align_up(p.off_rowstat + (size_t)N * 16, 1024);
  p.off_zt = align_up(p.off_shard + (size_t)N * 16, 1024);
  p.off_union = align_up(p.off_zt + (size_t)N * 4, 1024);
  const int64_t tiles_v = (V + BN - 1) / BN;
  p.fwd_bytes = (size_t)tiles_v * N * 8;
  if (p.off_union + p.fwd_bytes > budget) return false;
  const int64_t Vr = align_up((size_t)V, BN);
  double best = 1e300;
  bool found = false;
  for (int64_t nR = 1; nR <= 64; ++nR) {
    const int64_t R = (int64_t)align_up((size_t)((N + nR - 1) / nR), 256);
    if (nR > 1 && (nR - 1) * R >= N) continue;  // empty trailing block
    const size_t dx = align_up((size_t)R * H * 4, 1024);
    if (p.off_union + dx >= budget) continue;
    const size_t avail = budget - p.off_union - dx;
    int64_t Cv = (int64_t)(avail / ((size_t)R * 2)) / BN * BN;
    Cv = std::min(Cv, Vr);
    if (Cv < std::min<int64_t>(Vr, 1024)) continue;
    const int64_t nC = (V + Cv - 1) / Cv;
    const int64_t nRr = (N + R - 1) / R;
    // Cost model in bytes of extra HBM traffic: dW bf16 RMW per extra row block, dX fp32 RMW per
    // extra vocab chunk, and ~5 us of launch/tail per GEMM launch expressed as bytes at 6.5 TB/s.
    const double cost = (double)(nRr - 1) * V * H * 4 + (double)nRr * (nC - 1) * R * H * 8 +
                        (double)nRr * nC * 2 * 5e-6 * 6.5e12;
    if (cost < best) {
      best = cost;
      p.R = R;
      p.Cv = Cv;
      p.nR = nRr;
      p.nC = nC;
      found = true;
    }
  }
  if (!found) return false;
  const size_t g_bytes = align_up((size_t)p.R * p.Cv * 2, 1024);
  p.off_dxacc = p.off_union + g_bytes;
  p.bwd_bytes = g_bytes + (size_t)p.R * H * 4;
  p.total = p.off_union + std::max(p.fwd_bytes, p.bwd_bytes);
  if (p.total > budget) return false;
  *out = p;
  return true;
}

// Schedule S layout: header | sched arena | RowStat [N] | z_t [N] | row losses [N] | CSR counts
// [V+2] | CSR offsets [V+2] | hit rows [min(N,V)] | CSR token idx [N] | ShardStat [N] | stash
// reference [N] | row factor [N] | tile partials [tiles][2C] | stash [C][ld_stash] bf16.  C = the largest multiple of 256 rows that fits the budget.
bool plan_s(int64_t N, int64_t H, int64_t V, size_t budget, Plan* out) {
  if (N < 1 || H < 8 || V < 1) return false;
  if (budget == 0) budget = default_budget(N, V);
  Plan p;
  p.sched = SLF_SCHED_S;
  p.off_sched = WS_HEADER_BYTES;
  p.sched_bytes = sched_arena_bytes(N, H, V);
  p.off_rowstat = p.off_sched + p.sched_bytes;
  p.off_zt = align_up(p.off_rowstat + (size_t)N * 16, 1024);
  p.off_loss = align_up(p.off_zt + (size_t)N * 4, 1024);
  p.off_cnt = align_up(p.off_loss + (size_t)N * 4, 1024);
  p.off_off = align_up(p.off_cnt + (size_t)(V + 2) * 4, 1024);
  p.off_hits = align_up(p.off_off + (size_t)(V + 2) * 4, 1024);
  p.off_idx = align_up(p.off_hits + (size_t)std::min(N, V) * 4, 1024);
  p.off_shard = align_up(p.off_idx + (size_t)N * 4, 1024);  // per-chunk ShardStat (g = 1 path)
  p.off_mref = align_up(p.off_shard + (size_t)N * 16, 1024);
  p.off_fac = align_up(p.off_mref + (size_t)N * 4, 1024);
  p.off_part = align_up(p.off_fac + (size_t)N * 4, 1024);
  const int64_t tiles_v = (V + BN - 1) / BN;
  p.ld_stash = (int64_t)align_up((size_t)V, 8);
  const int64_t Nmax = (int64_t)align_up((size_t)N, 256);
  int64_t best = 0;
  for (int64_t C = 256; C <= Nmax; C += 256) {
    const size_t part = align_up((size_t)tiles_v * 2 * C * 8, 1024);  // 2C: room for extended chunks
    const size_t tot = p.off_part + part + (size_t)C * p.ld_stash * 2 + 256;
    if (tot <= budget) best = C;
    else break;
  }
  if (best == 0) return false;
  p.C = best;
  p.nCh = (N + best - 1) / best;
  p.off_stash = p.off_part + align_up((size_t)tiles_v * 2 * best * 8, 1024);
  p.total = p.off_stash + (size_t)best * p.ld_stash * 2 + 256;  // tail pad: 3-D stash loads over-read < 128 B
  p.fwd_bytes = p.total - p.off_part;
  *out = p;
  return true;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

slf_status check_common(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                        int64_t V, const void* ws) {
  if (!hidden || !weight || !targets || !ws) return fail(SLF_ERR_ARG, "null required pointer");
  if (N < 1 || H < 8 || V < 1) return fail(SLF_ERR_ARG, "bad sizes N=%lld H=%lld V=%lld", (long long)N, (long long)H, (long long)V);
  if (H % 8) return fail(SLF_ERR_ARG, "H must be a multiple of 8 (got %lld)", (long long)H);
  if (N > (1ll << 31) - 1 || V > (1ll << 31) - 1 || H > (1 << 20)) return fail(SLF_ERR_ARG, "sizes exceed int32 tile indexing");
  if (!aligned16(hidden) || !aligned16(weight) || !aligned16(targets) || !aligned16(ws))
    return fail(SLF_ERR_ALIGN, "device pointers must be 16-byte aligned");
  return SLF_OK;
}

// ---- phases ------------------------------------------------------------------------------------
struct Ctx {
  DevInfo* dev;
  cudaStream_t s;
  uint8_t* ws;
  Plan plan;
  bool acc_dw = false;  // SLF_FLAG_ACCUMULATE_DW: dW += instead of dW =
  const cudaEvent_t* chunk_ready = nullptr;  // schedule S: chunk k's hidden rows are on the device
  // schedule S: enqueues the chunked input copies once this call's own small H2D copies (targets,
  // tile tables) are queued — copies share the H2D engine in FIFO order
  std::function<slf_status()> enqueue_inputs;
  std::function<slf_status()> after_prep;  // e.g. the data-parallel all-reduce of n_valid
  int cj_red = SLF_MEAN;  // reduction / scale of the call, for the stash epilogue's rescale bound
  float cj_scale = 1.f;
};

WsHeader* hdr_of(uint8_t* ws) { return reinterpret_cast<WsHeader*>(ws); }
double* block_sums_of(uint8_t* ws) { return reinterpret_cast<double*>(ws + 256); }

// Per-call arena of LPT tile tables (uploaded once per call into the workspace).
// LPT tables depend only on the problems' tile counts, K and epilogue kinds: memoised across calls
// (building one is O(tiles x units) on the host, ~0.5 ms at the Llama-8B group shape).
struct LptCache {
  std::mutex mu;
  std::map<std::vector<int64_t>, std::pair<std::vector<int>, int>> m;
};
LptCache g_lpt;

std::vector<int> lpt_table_cached(const ProbSpec* ps, int n, int units, int* stride) {
  std::vector<int64_t> key{units, n};
  for (int p = 0; p < n; ++p)
    key.insert(key.end(), {ps[p].a.M, ps[p].a.N, ps[p].a.K, ps[p].a.num_tiles, ps[p].epi, ps[p].a.mode});
  std::lock_guard<std::mutex> lk(g_lpt.mu);
  auto it = g_lpt.m.find(key);
  if (it == g_lpt.m.end()) {
    if (g_lpt.m.size() >= 256) g_lpt.m.clear();
    int st = 0;
    std::vector<int> t = lpt_table(ps, n, units, &st);
    it = g_lpt.m.emplace(key, std::make_pair(std::move(t), st)).first;
  }
  *stride = it->second.second;
  return it->second.first;  // a copy, taken under the lock
}

// Pinned copies of tile tables referenced by captured CUDA graphs (content-keyed, never freed).
const uint8_t* captured_table(const std::vector<int>& host, size_t bytes) {
  static std::vector<std::pair<std::vector<int>, uint8_t*>> pool;
  for (auto& e : pool)
    if (e.first == host) return e.second;
  uint8_t* p = nullptr;
  // the allocation is not a stream operation: relaxed capture mode for this thread while it runs
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  const cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), bytes, cudaHostAllocDefault);
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) return nullptr;
  memcpy(p, host.data(), bytes);
  pool.emplace_back(host, p);
  return p;
}

struct SchedArena {
  std::vector<int> host;
  std::vector<std::pair<size_t, int>> tables;  // (offset in ints, stride)
  int add(const ProbSpec* ps, int n, int units) {
    int stride = 0;
    const std::vector<int> t = lpt_table_cached(ps, n, units, &stride);
    tables.push_back({host.size(), stride});
    host.insert(host.end(), t.begin(), t.end());
    return (int)tables.size() - 1;
  }
  bool fits(const Ctx& c) const { return host.size() * 4 <= c.plan.sched_bytes; }
  slf_status upload(Ctx& c) {
    if (host.empty()) return SLF_OK;
    if (!fits(c)) return fail(SLF_ERR_WORKSPACE, "tile schedule arena overflow");
    const size_t bytes = host.size() * 4;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    SLF_CUDA(cudaStreamIsCapturing(c.s, &cap));
    if (cap == cudaStreamCaptureStatusActive) {
      // CUDA-graph capture: the copy becomes a graph node that reads its host source at every
      // replay, so the source must outlive the graph and never change — a pinned buffer per
      // distinct table content, kept for the life of the process (no events: a capture cannot
      // wait on the ring's).
      const uint8_t* src = captured_table(host, bytes);
      if (!src) return fail(SLF_ERR_CUDA, "cannot allocate pinned memory for a captured tile table");
      SLF_CUDA(cudaMemcpyAsync(c.ws + c.plan.off_sched, src, bytes, cudaMemcpyHostToDevice, c.s));
      return SLF_OK;
    }
    PinnedRing& r = c.dev->ring;
    if (!r.buf) {
      SLF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&r.buf), (size_t)RING_SLOTS * SCHED_ARENA_MAX,
                             cudaHostAllocDefault));
      for (int i = 0; i < RING_SLOTS; ++i) SLF_CUDA(cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming));
    }
    const int k = r.next;
    r.next = (r.next + 1) % RING_SLOTS;
    if (r.used[k]) SLF_CUDA(cudaEventSynchronize(r.ev[k]));
    uint8_t* slot = r.buf + (size_t)k * SCHED_ARENA_MAX;
    memcpy(slot, host.data(), bytes);
    SLF_CUDA(cudaMemcpyAsync(c.ws + c.plan.off_sched, slot, bytes, cudaMemcpyHostToDevice, c.s));
    SLF_CUDA(cudaEventRecord(r.ev[k], c.s));
    r.used[k] = true;
    return SLF_OK;
  }
  const int* dev(Ctx& c, int k) const {
    return reinterpret_cast<const int*>(c.ws + c.plan.off_sched) + tables[k].first;
  }
};

// Forward statistics of one shard: EPI_STATS GEMM over all (row tile, vocab tile), then the
// per-row merge into ShardStat.
slf_status phase_stats(Ctx& c, const void* X, const void* W, const int32_t* t, int64_t N, int64_t H, int64_t V_l,
                       int64_t vocab_start, int32_t ignore_index, slf_shardstat* out) {
  CUtensorMap ta, tb;
  SLF_TRY(tmap_kmajor(&ta, X, H, N, H, BM));
  SLF_TRY(tmap_kmajor(&tb, W, H, V_l, H, b_box_rows()));
  GemmArgs a{};
  a.M = (int)N;
  a.N = (int)V_l;
  a.K = (int)H;
  a.targets = t;
  a.tcol0 = vocab_start;
  a.ignore_index = ignore_index;
  a.partials = reinterpret_cast<float2*>(c.ws + c.plan.off_union);
  a.zt = reinterpret_cast<float*>(c.ws + c.plan.off_zt);
  SLF_TRY((launch_gemm<EPI_STATS, false, false>(c.dev, ta, tb, a, c.s)));
  const int tiles_v = (int)((V_l + BN - 1) / BN);
  ProfScope ps(SLF_PROF_LOCAL_COMBINE, c.s, 0.0, (double)N * (tiles_v * 8.0 + 4 + 4 + 16));
  local_combine_kernel<<<(unsigned)((N + 255) / 256), 256, 0, c.s>>>(a.partials, tiles_v, a.zt, t, N, vocab_start,
                                                                     V_l, ignore_index, out);
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

slf_status launch_prep(Ctx& c, const int32_t* t, int64_t N, int32_t ignore_index, int64_t V_global) {
  ProfScope ps(SLF_PROF_PREP, c.s, 0.0, (double)N * 4);
  prep_targets_kernel<<<1, 1024, 0, c.s>>>(t, N, ignore_index, V_global, hdr_of(c.ws));
  SLF_CUDA(cudaGetLastError());
  if (c.after_prep) SLF_TRY(c.after_prep());
  return SLF_OK;
}

slf_status phase_combine(Ctx& c, const slf_shardstat* st, int g, const int32_t* t, int64_t N, int64_t vocab_start,
                         int64_t V_l, int64_t V_global, int32_t ignore_index, int reduction, float scale,
                         float* loss_out, slf_rowstat* rowstat) {
  const unsigned blocks = (unsigned)((N + 255) / 256);
  if (blocks > (unsigned)MAX_LOSS_BLOCKS)
    return fail(SLF_ERR_ARG, "N = %lld too large for the loss reduction (at most %lld rows)", (long long)N,
                (long long)MAX_LOSS_BLOCKS * 256);
  SLF_TRY(launch_prep(c, t, N, ignore_index, V_global));
  ProfScope ps(SLF_PROF_FINAL_COMBINE, c.s, 0.0, (double)N * (g * 16.0 + 4 + 16 + 4));
  final_combine_kernel<<<blocks, 256, 0, c.s>>>(st, g, t, N, vocab_start, V_l, V_global, ignore_index, reduction,
                                                scale, loss_out, rowstat, hdr_of(c.ws), block_sums_of(c.ws));
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

// Backward (schedule R): for each row block r, for each vocab chunk c: recompute the logits tile
// by tile and form G (EPI_GRAD), then ONE grouped launch of dW_c (+)= G^T X_r (EPI_DW) and
// dX_r (+)= G W_c (EPI_DX) with an LPT tile table (no wave quantisation between the two).
slf_status phase_backward(Ctx& c, const void* X, const void* W, const slf_rowstat* rowstat, int64_t N, int64_t H,
                          int64_t V_l, float grad_scale, void* dX, int dX_fp32, void* dW) {
  if (!dX && !dW) return SLF_OK;
  const Plan& p = c.plan;
  uint8_t* G = c.ws + p.off_union;
  float* dxacc = reinterpret_cast<float*>(c.ws + p.off_dxacc);
  const int64_t ldG = p.Cv;
  const int cg = cta_group();
  const int units = c.dev->sms / cg;

  auto build = [&](int64_t rb, int64_t cb, ProbSpec* ps, int* n) -> slf_status {
    const int64_t r0 = rb * p.R, rows = std::min(p.R, N - r0);
    const int64_t c0 = cb * p.Cv, wc = std::min(p.Cv, V_l - c0);
    const uint8_t* Xr = reinterpret_cast<const uint8_t*>(X) + (size_t)r0 * H * 2;
    const uint8_t* Wc = reinterpret_cast<const uint8_t*>(W) + (size_t)c0 * H * 2;
    *n = 0;
    if (dW) {  // dW[c0:c0+wc] (+)= G^T X_r : A = G^T (MN-major), B = X_r (MN-major)
      ProbSpec& q = ps[(*n)++];
      SLF_TRY(tmap_mnmajor(&q.ta, G, wc, rows, ldG));
      SLF_TRY(tmap_mnmajor(&q.tb, Xr, H, rows, H, b_box_rows() / 64));
      q.epi = EPI_DW;
      q.a_mn = q.b_mn = true;
      q.a = GemmArgs{};
      q.a.M = (int)wc;
      q.a.N = (int)H;
      q.a.K = (int)rows;
      q.a.out = reinterpret_cast<uint8_t*>(dW) + (size_t)c0 * H * 2;
      q.a.ld_out = H;
      q.a.mode = (rb > 0 || c.acc_dw) ? dw_acc_mode() : 0;
      SLF_TRY(tmap_kmajor(&q.tc, q.a.out, H, wc, H, BM));
      finish_geometry(q.a, cg);
    }
    if (dX) {  // dX_r (+)= G W_c : A = G (K-major), B = W_c (MN-major)
      ProbSpec& q = ps[(*n)++];
      SLF_TRY(tmap_kmajor(&q.ta, G, wc, rows, ldG, BM));
      SLF_TRY(tmap_mnmajor(&q.tb, Wc, H, wc, H, b_box_rows() / 64));
      q.epi = EPI_DX;
      q.a_mn = false;
      q.b_mn = true;
      GemmArgs a{};
      a.M = (int)rows;
      a.N = (int)H;
      a.K = (int)wc;
      a.rowstat = rowstat + r0;
      if (dX_fp32) {
        a.out = reinterpret_cast<float*>(dX) + (size_t)r0 * H;
        a.ld_out = H;
        a.mode = cb == 0 ? DX_STORE_F32 : DX_ACC_F32;
      } else {
        a.out = dxacc;
        a.ld_out = H;
        a.out2 = reinterpret_cast<uint8_t*>(dX) + (size_t)r0 * H * 2;
        a.ld_out2 = H;
        a.mode = p.nC == 1 ? DX_STORE_FINAL_BF16
                 : cb == 0 ? DX_STORE_F32
                 : cb == p.nC - 1 ? DX_ACC_FINAL_BF16
                                  : DX_ACC_F32;
      }
      finish_geometry(a, cg);
      q.a = a;
    }
    return SLF_OK;
  };

  // LPT tables for the (at most 4) distinct (rows, wc) shapes, uploaded once.
  SchedArena arena;
  std::vector<std::pair<std::pair<int64_t, int64_t>, int>> keys;
  for (int64_t rb = 0; rb < p.nR; ++rb)
    for (int64_t cb = 0; cb < p.nC; ++cb) {
      const auto key = std::make_pair(std::min(p.R, N - rb * p.R), std::min(p.Cv, V_l - cb * p.Cv));
      bool have = false;
      for (auto& k : keys) have |= k.first == key;
      if (have) continue;
      ProbSpec ps[2];
      int n = 0;
      SLF_TRY(build(rb, cb, ps, &n));
      keys.push_back({key, arena.add(ps, n, units)});
    }
  SLF_TRY(arena.upload(c));

  for (int64_t rb = 0; rb < p.nR; ++rb) {
    const int64_t r0 = rb * p.R;
    const int64_t rows = std::min(p.R, N - r0);
    if (rows <= 0) break;
    const uint8_t* Xr = reinterpret_cast<const uint8_t*>(X) + (size_t)r0 * H * 2;
    for (int64_t cb = 0; cb < p.nC; ++cb) {
      const int64_t c0 = cb * p.Cv;
      const int64_t wc = std::min(p.Cv, V_l - c0);
      const uint8_t* Wc = reinterpret_cast<const uint8_t*>(W) + (size_t)c0 * H * 2;
      {  // G[rows, wc] = coef * (softmax - onehot), recomputed
        CUtensorMap ta, tb;
        SLF_TRY(tmap_kmajor(&ta, Xr, H, rows, H, BM));
        SLF_TRY(tmap_kmajor(&tb, Wc, H, wc, H, b_box_rows()));
        GemmArgs a{};
        a.M = (int)rows;
        a.N = (int)wc;
        a.K = (int)H;
        a.rowstat = rowstat + r0;
        a.col0 = c0;
        a.grad_scale = grad_scale;
        a.out = G;
        a.ld_out = ldG;
        a.rows_buf = (int)p.R;
        SLF_TRY((launch_gemm<EPI_GRAD, false, false>(c.dev, ta, tb, a, c.s)));
      }
      ProbSpec ps[2];
      int n = 0;
      SLF_TRY(build(rb, cb, ps, &n));
      int k = 0;
      const auto key = std::make_pair(rows, wc);
      for (auto& kk : keys)
        if (kk.first == key) k = kk.second;
      SLF_TRY(launch_group(c.dev, ps, n, c.s, arena.dev(c, k), arena.tables[k].second,
                           n == 2 ? SLF_PROF_GEMM_GROUP : -1));
    }
  }
  return SLF_OK;
}

// ---- schedule S ---------------------------------------------------------------------------------
// Per row chunk, ONE forward GEMM whose epilogue keeps the tile statistics and stashes
// p~ = bf16(exp(z - m_tile)); the g shards' row statistics are merged and the stash is rescaled in
// place into the softmax term G_P; ONE grouped launch of dX_chunk = G_P W (- coef W[t], exact, in
// the epilogue) and dW (+)= G_P^T X_chunk; finally dW[v] -= coef sum_{t_i = v} x_i from the target
// CSR.  No logits are recomputed: 6 N H V tensor FLOPs.  The pieces below are used by the fused
// single-GPU call (g = 1) and by the vocab-shard split API (the caller gathers the per-chunk
// statistics and all-reduces the per-chunk fp32 dX partials).
struct SArgs {
  const void* X;
  const void* W;  // this shard's rows [vocab_start, vocab_start + V_l)
  const int32_t* t;
  int64_t N, H, V_l, vs, Vg;
  int32_t ign;
};

// Target CSR of the shard: counts (integer atomics: order-free) -> exclusive
// scan (offsets, hit rows) -> stable rank -> scatter.  The stable rank sorts blocks of 4096 tokens
// by packed (target, token) keys in `scratch` (>= round_up(N, 4096) * 4 bytes) and binary-searches
// them; without that much scratch it falls back to the brute-force rank.  `bsum` (>= 8 bytes per
// 8192 vocabulary rows, or null) holds the multi-block scan's span totals.
size_t csr_sort_bytes(int64_t N) { return (size_t)((N + CSR_SORT_T - 1) / CSR_SORT_T) * CSR_SORT_T * 4; }

slf_status build_csr(cudaStream_t st, const int32_t* t, int64_t N, int32_t ign, int64_t vs, int64_t V_l, int32_t* cnt,
                     int32_t* off, int32_t* hits, int32_t* idx, int2* bsum, size_t bsum_bytes, uint8_t* scratch,
                     size_t scratch_bytes) {
  ProfScope ps(SLF_PROF_CSR, st, 0.0, (double)V_l * 12 + (double)N * 12);
  csr_zero_kernel<<<(unsigned)std::min<int64_t>((V_l + 2 + 255) / 256, 1024), 256, 0, st>>>(cnt, V_l + 2);
  csr_count_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(t, N, ign, vs, V_l, cnt);
  const int64_t nspan = (V_l + CSR_SCAN_SPAN - 1) / CSR_SCAN_SPAN;
  if (nspan > 1 && bsum && (size_t)nspan * 8 <= bsum_bytes) {
    csr_blocksum_kernel<<<(unsigned)nspan, 1024, 0, st>>>(cnt, V_l, bsum);
    csr_scan_kernel<<<(unsigned)nspan, 1024, 0, st>>>(cnt, V_l, off, hits, bsum);
  } else {
    csr_scan_kernel<<<1, 1024, 0, st>>>(cnt, V_l, off, hits);
  }
  static const bool brute = getenv("SLF_CSR_BRUTE") != nullptr;  // A/B knob: the round-1 rank
  if (!brute && scratch && scratch_bytes >= csr_sort_bytes(N) && V_l < (1 << (32 - CSR_SORT_SHIFT))) {
    uint32_t* sorted = reinterpret_cast<uint32_t*>(scratch);
    csr_block_sort_kernel<<<(unsigned)((N + CSR_SORT_T - 1) / CSR_SORT_T), 1024, 0, st>>>(t, N, ign, vs, V_l, sorted);
    csr_rank_scatter_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(t, N, ign, vs, V_l, cnt, off, sorted, idx);
  } else {
    csr_scatter_kernel<<<(unsigned)((N + CSR_TOK_PER_BLOCK - 1) / CSR_TOK_PER_BLOCK), 256, 0, st>>>(t, N, ign, vs,
                                                                                                  V_l, cnt, off, idx);
  }
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

slf_status s_begin(Ctx& c, const SArgs& a, bool need_dw) {
  const Plan& p = c.plan;
  SLF_CUDA(cudaMemsetAsync(c.ws + WS_SYNC_OFF, 0, WS_SYNC_BYTES, c.s));  // in-kernel combine sync words
  SLF_TRY(launch_prep(c, a.t, a.N, a.ign, a.Vg));
  if (need_dw) {
    // scratch: the tile-partials + stash region, idle until the first chunk's stash GEMM; span
    // totals in the (idle) ShardStat area
    SLF_TRY(build_csr(c.s, a.t, a.N, a.ign, a.vs, a.V_l, reinterpret_cast<int32_t*>(c.ws + p.off_cnt),
                      reinterpret_cast<int32_t*>(c.ws + p.off_off), reinterpret_cast<int32_t*>(c.ws + p.off_hits),
                      reinterpret_cast<int32_t*>(c.ws + p.off_idx), reinterpret_cast<int2*>(c.ws + p.off_shard),
                      (size_t)a.N * 16, c.ws + p.off_part, p.total - p.off_part));
  }
  return SLF_OK;
}

// Stash GEMM of chunk `ch` and this shard's per-row statistics of the chunk (out[rows]).
// One row chunk of schedule S: rows [r0, r0 + rows).  The first min(rows, C) stash rows live in the
// workspace; on the fused single-GPU call the chunk may be extended by `ext` rows whose stash
// lives in the caller's dhidden buffer beyond this chunk's rows (rows not written yet).
struct SChunk {
  int64_t index, r0, rows, ext;
  uint8_t* ext_base;  // stash rows [rows - ext, rows): row stride ld_stash, or nullptr
  uint8_t* xt = nullptr;  // X_chunk^T [H][ld_xt] (dW's B operand K-major) in free dhidden rows, or nullptr
  int64_t ld_xt = 0;
  const uint8_t* xrows = nullptr;  // the chunk's hidden rows when not X + r0 (fused RMSNorm: its y buffer)
  bool ref = false;       // per-row stash reference; false: the stash is rescaled in place
  uint8_t* xs = nullptr;  // with ref and dW: X'_chunk = bf16(f ⊙ X) [rows][H], the dW GEMM's B operand
  // Vocab-sharded call only (shard_chunks): where the chunk's fp32 dX partial lives — a byte offset
  // into dhidden (>= 0), PART_WS_TAIL (the workspace stash's tail) or PART_WS_REGION (a dedicated
  // workspace region) — and the end (bytes into dhidden) of the rows X'^T may use.
  int64_t part_off = -1;
  size_t xt_lim = 0;
  bool cj = false;  // the chunk's combine runs inside its group launch (CombineJob)
};
constexpr int64_t PART_WS_TAIL = -1, PART_WS_REGION = -2;

SChunk s_plain_chunk(const Plan& p, int64_t N, int64_t ch) {
  const int64_t r0 = ch * p.C;
  return SChunk{ch, r0, std::min(p.C, N - r0), 0, nullptr, nullptr, 0};
}

// X_chunk^T for the dW GEMM's K-major B operand (programmatic dependent launch).
slf_status launch_transpose_x(Ctx& c, const SArgs& a, const SChunk& k) {
  ProfScope ps(SLF_PROF_TRANSPOSE, c.s, 0.0, (double)k.rows * a.H * 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((k.rows + 63) / 64), (unsigned)((a.H + 63) / 64));
  cfg.blockDim = dim3(256);
  cfg.stream = c.s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SLF_CUDA(cudaLaunchKernelEx(&cfg, transpose_x_kernel,
                              reinterpret_cast<const uint16_t*>(a.X) + (size_t)k.r0 * a.H, a.H, (int)k.rows,
                              reinterpret_cast<uint16_t*>(k.xt), k.ld_xt));
  return SLF_OK;
}

// Stash GEMM of a chunk and this shard's per-row statistics of the chunk (out[rows]).
slf_status s_chunk_stats(Ctx& c, const SArgs& a, const SChunk& k, slf_shardstat* out) {
  const Plan& p = c.plan;
  const int64_t r0 = k.r0, rows = k.rows, main_rows = rows - k.ext;
  float* zt = reinterpret_cast<float*>(c.ws + p.off_zt);
  float2* part = reinterpret_cast<float2*>(c.ws + p.off_part);
  ProbSpec ps;
  const uint8_t* Xr = k.xrows ? k.xrows : reinterpret_cast<const uint8_t*>(a.X) + (size_t)r0 * a.H * 2;
  SLF_TRY(tmap_kmajor(&ps.ta, Xr, a.H, rows, a.H, BM));
  SLF_TRY(tmap_kmajor(&ps.tb, a.W, a.H, a.V_l, a.H, b_box_rows()));
  GemmArgs g{};
  g.M = (int)rows;
  g.N = (int)a.V_l;
  g.K = (int)a.H;
  g.targets = a.t + r0;
  g.tcol0 = a.vs;
  g.ignore_index = a.ign;
  g.partials = part;
  g.zt = zt + r0;
  g.out = c.ws + p.off_stash;
  g.ld_out = p.ld_stash;
  if (k.ref) g.mref = reinterpret_cast<const float*>(c.ws + p.off_mref) + r0;
  static const int dbg = getenv("SLF_DEBUG_EPI") ? atoi(getenv("SLF_DEBUG_EPI")) : 0;
  g.mode = (dbg & 64) ? 32 : 0;  // timing experiment only (SLF_DEBUG_EPI=64): skip the stash stores
  g.tma_out = 1;      // the stash is written through TMA-staged stores
  SLF_TRY(tmap_kmajor(&ps.tc, c.ws + p.off_stash, a.V_l, main_rows, p.ld_stash, BM));
  if (k.ext) {
    SLF_TRY(tmap_kmajor(&ps.tc2, k.ext_base, a.V_l, k.ext, p.ld_stash, BM));
    ps.c_split = (int)main_rows;
  }
  if (k.cj) {  // the group launch's dX tiles may start before the combine: flag possible rescales
    g.fb_flag = reinterpret_cast<unsigned*>(c.ws + WS_SYNC_OFF) + 2 * k.index + 1;
    g.fb_hdr = hdr_of(c.ws);
    g.fb_red = c.cj_red;
    g.fb_scale = c.cj_scale;
    g.fb_gscale = 1.0f;
  }
  ps.a = g;
  ps.epi = EPI_STASH;
  // The mainloop may start before the previous grid completes (GroupArgs::early) when its operands
  // are the caller's hidden rows and W, which nothing in the call writes — and only from the second
  // chunk on: a kernel of ours just before the call (e.g. rmsnorm_fwd producing the hidden rows)
  // triggers its dependents early, so the first GEMM of a call must wait; a later chunk's stash GEMM
  // launches only once the previous group launch is fully resident, i.e. after every earlier grid
  // completed.  Host-input calls: not while chunks wait for their rows' copies (chunks 0-2).
  ps.ro_operands = k.xrows == nullptr && k.index >= 1 && !(c.chunk_ready && k.index <= 2);
  SLF_TRY(launch_group(c.dev, &ps, 1, c.s));
  if (out) {  // shard statistics for the all-gather (vocab shards); one GPU merges in combine_transform
    const int tiles_v = (int)((a.V_l + BN - 1) / BN);
    ProfScope pr(SLF_PROF_LOCAL_COMBINE, c.s, 0.0, (double)rows * (tiles_v * 8.0 + 24));
    shard_rows_tpr_kernel<<<(unsigned)((rows + SR_ROWS - 1) / SR_ROWS), 256, 0, c.s>>>(
        part, tiles_v, (int)rows, zt + r0, a.t + r0, a.vs, a.V_l, a.ign, out);
    SLF_CUDA(cudaGetLastError());
  }
  return SLF_OK;
}

slf_status s_build_bwd(Ctx& c, const SArgs& a, const SChunk& k, void* dXc, int dx_fp32, void* dW, ProbSpec* ps,
                       int* n) {
  const Plan& p = c.plan;
  const int cg = cta_group();
  const int64_t r0 = k.r0, rows = k.rows, main_rows = rows - k.ext;
  const uint8_t* Xr = k.xrows ? k.xrows : reinterpret_cast<const uint8_t*>(a.X) + (size_t)r0 * a.H * 2;
  uint8_t* stash = c.ws + p.off_stash;
  slf_rowstat* rs = reinterpret_cast<slf_rowstat*>(c.ws + p.off_rowstat);
  *n = 0;
  if (dXc) {  // dX_chunk = G_P W : A = G_P (K-major over V_l, rows split ws | ext), B = W (MN-major)
    ProbSpec& q = ps[(*n)++];
    q = ProbSpec{};
    SLF_TRY(tmap_kmajor(&q.ta, stash, a.V_l, main_rows, p.ld_stash, BM));
    if (k.ext) {
      SLF_TRY(tmap_kmajor(&q.ta2, k.ext_base, a.V_l, k.ext, p.ld_stash, BM));
      q.a_split = (int)main_rows;
    }
    SLF_TRY(tmap_mnmajor(&q.tb, a.W, a.H, a.V_l, a.H, b_box_rows() / 64));
    q.epi = EPI_DXS;
    q.a_mn = false;
    q.b_mn = true;
    q.a.M = (int)rows;
    q.a.N = (int)a.H;
    q.a.K = (int)a.V_l;
    q.a.rowstat = rs + r0;
    q.a.grad_scale = 1.0f;
    q.a.wrow = reinterpret_cast<const uint16_t*>(a.W);
    q.a.ld_w = a.H;
    q.a.out = dXc;
    q.a.ld_out = a.H;
    q.a.mode = dx_fp32 ? 1 : 0;
    if (k.ref) q.a.fac = reinterpret_cast<const float*>(c.ws + p.off_fac) + r0;
    finish_geometry(q.a, cg);
  }
  if (dW) {  // dW (+)= G_P^T X_chunk : A = G_P^T (MN-major; K = rows split ws | ext), B = X_chunk (MN-major)
    ProbSpec& q = ps[(*n)++];
    q = ProbSpec{};
    if (!k.ext && a.V_l % 64 && mn3d_enabled()) {
      // The workspace stash (no second segment): a 3-D map even when V_l % 64 != 0 (e.g. 16032
      // vocabulary rows per rank at g = 8).  Its last atom reads up to 63 columns past V_l — rows
      // >= M of the A operand, whose products only reach dW rows >= V_l, which the store map
      // clips; past the last stash row it reads into the workspace's 256-byte tail pad.
      SLF_TRY(make_tmap_mn3d(&q.ta, stash, (uint64_t)a.V_l, (uint64_t)main_rows, (uint64_t)p.ld_stash * 2, 2));
      q.a3d_force = true;
    } else {
      SLF_TRY(tmap_mnmajor(&q.ta, stash, a.V_l, main_rows, p.ld_stash));
    }
    if (k.ext) {
      SLF_TRY(tmap_mnmajor(&q.ta2, k.ext_base, a.V_l, k.ext, p.ld_stash));
      q.a_split = (int)main_rows;
    }
    q.epi = EPI_DW;
    q.a_mn = true;
    if (k.xt) {  // B = X_chunk^T [H][ld_xt]: K-major
      SLF_TRY(tmap_kmajor(&q.tb, k.xt, rows, a.H, k.ld_xt, b_box_rows()));
      q.b_mn = false;
    } else {
      SLF_TRY(tmap_mnmajor(&q.tb, k.xs ? k.xs : Xr, a.H, rows, a.H, b_box_rows() / 64));
      q.b_mn = true;
    }
    q.a.M = (int)a.V_l;
    q.a.N = (int)a.H;
    q.a.K = (int)rows;
    q.a.out = dW;
    q.a.ld_out = a.H;
    q.a.mode = (k.index > 0 || c.acc_dw) ? dw_acc_mode() : 0;
    static const bool no_rmw = getenv("SLF_DEBUG_DW_NO_RMW") != nullptr;  // timing experiments only (wrong dW)
    if (no_rmw) q.a.mode = 0;
    SLF_TRY(tmap_kmajor(&q.tc, dW, a.H, a.V_l, a.H, BM));
    finish_geometry(q.a, cg);
  }
  return SLF_OK;
}

// Merge the g shards' statistics of the chunk (st[g][rows], shard order; nullptr on one GPU: the
// chunk's own tile partials), transform the stash in place, and run the grouped dX/dW launch.
// dXc = row 0 of the chunk's dhidden rows (bf16, or fp32 when dx_fp32: this shard's partial, to be
// summed across shards).  `sched` (optional) is a prebuilt LPT table for this chunk shape.
slf_status s_chunk_bwd(Ctx& c, const SArgs& a, const SChunk& k, const slf_shardstat* st, int g, int reduction,
                       float scale, float* loss_rows_all, void* dXc, int dx_fp32, void* dW, const int* sched = nullptr,
                       int sched_stride = 0, const RmsStep* rms = nullptr) {
  const Plan& p = c.plan;
  const int64_t r0 = k.r0, rows = k.rows;
  const int tiles_v = (int)((a.V_l + BN - 1) / BN);
  static const bool skip_ct = getenv("SLF_DEBUG_EPI") && (atoi(getenv("SLF_DEBUG_EPI")) & 512);  // timing only
  // SLF_DEBUG_CT2=1 (timing only): the combine launch is issued twice (same outputs) — its exposed
  // cost per chunk is the step-time difference
  static const int ct_reps = getenv("SLF_DEBUG_CT2") && atoi(getenv("SLF_DEBUG_CT2")) == 1 ? 2 : 1;
  // In-kernel combine (k.cj): the group launch's epilogue warps do the work of combine_scale_kernel
  // below, and its dX tiles start on the stash without waiting for it
  CombineJob cj{};
  const bool in_kernel = k.cj && !skip_ct && !rms && !st && g == 1 && (dXc || dW);
  if (in_kernel) {
    cj.partials = reinterpret_cast<const float2*>(c.ws + p.off_part);
    cj.zt = reinterpret_cast<const float*>(c.ws + p.off_zt) + r0;
    cj.t = a.t + r0;
    cj.mref = reinterpret_cast<const float*>(c.ws + p.off_mref) + r0;
    cj.hdr = hdr_of(c.ws);
    cj.loss_rows = loss_rows_all + r0;
    cj.rowstat = reinterpret_cast<slf_rowstat*>(c.ws + p.off_rowstat) + r0;
    cj.fac = reinterpret_cast<float*>(c.ws + p.off_fac) + r0;
    cj.stash = reinterpret_cast<uint16_t*>(c.ws + p.off_stash);
    cj.stash2 = reinterpret_cast<uint16_t*>(k.ext_base);
    cj.xrows = reinterpret_cast<const uint16_t*>(k.xrows ? k.xrows
                                                         : reinterpret_cast<const uint8_t*>(a.X) + (size_t)r0 * a.H * 2);
    cj.xs = reinterpret_cast<uint16_t*>(k.xt);
    cj.V_l = a.V_l;
    cj.ld_stash = p.ld_stash;
    cj.H = a.H;
    cj.ld_xst = k.xt ? k.ld_xt : 0;
    cj.tiles = tiles_v;
    cj.rows = (int)rows;
    cj.split = (int)(rows - k.ext);
    cj.reduction = reduction;
    cj.ign = a.ign;
    cj.scale = scale;
    cj.grad_scale = 1.0f;
    cj.counter = reinterpret_cast<unsigned*>(c.ws + WS_SYNC_OFF) + 2 * k.index;
    cj.fb_flag = cj.counter + 1;
  }
  if (in_kernel) {
  } else if (k.ref && !skip_ct) {  // per-row stash reference: factors and X'_chunk, the stash stays as is
    ProfScope ps(SLF_PROF_COMBINE_TRANSFORM, c.s, 0.0, (double)rows * (tiles_v * 8.0 + a.H * 4.0 + 40.0));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((rows + CS_ROWS - 1) / CS_ROWS + (rms ? rms_blocks_of(*rms) : 0)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = tiles_v * sizeof(float);
    cfg.stream = c.s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint8_t* xr = k.xrows ? k.xrows : reinterpret_cast<const uint8_t*>(a.X) + (size_t)r0 * a.H * 2;
    for (int rep = 0; rep < (rms ? 1 : ct_reps); ++rep)
    SLF_CUDA(cudaLaunchKernelEx(
        &cfg, combine_scale_kernel, reinterpret_cast<const float2*>(c.ws + p.off_part), tiles_v, (int)rows,
        reinterpret_cast<const float*>(c.ws + p.off_zt) + r0, a.t + r0, a.V_l, p.ld_stash, a.ign, reduction, scale, 1.0f,
        (const WsHeader*)hdr_of(c.ws), loss_rows_all + r0, reinterpret_cast<slf_rowstat*>(c.ws + p.off_rowstat) + r0,
        reinterpret_cast<uint16_t*>(c.ws + p.off_stash), reinterpret_cast<uint16_t*>(k.ext_base), (int)(rows - k.ext),
        reinterpret_cast<const float*>(c.ws + p.off_mref) + r0, reinterpret_cast<float*>(c.ws + p.off_fac) + r0,
        reinterpret_cast<const uint16_t*>(xr), reinterpret_cast<uint16_t*>(k.xt ? k.xt : k.xs), a.H,
        k.xt ? k.ld_xt : 0, rms ? *rms : RmsStep{}, st, g, a.vs, a.Vg));
  } else if (!skip_ct) {
    ProfScope ps(SLF_PROF_COMBINE_TRANSFORM, c.s, 0.0, (double)rows * (tiles_v * 8.0 + a.V_l * 4.0 + 16.0 * g + 24));
    // Programmatic dependent launch: blocks start while the stash GEMM drains and wait in-kernel.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(rows + (rms ? rms_blocks_of(*rms) : 0)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = tiles_v * sizeof(float);
    cfg.stream = c.s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SLF_CUDA(cudaLaunchKernelEx(
        &cfg, combine_transform_kernel, st, g, reinterpret_cast<const float2*>(c.ws + p.off_part), tiles_v, (int)rows,
        reinterpret_cast<const float*>(c.ws + p.off_zt) + r0, a.t + r0, a.vs, a.V_l, a.Vg, p.ld_stash, a.ign,
        reduction, scale, 1.0f, (const WsHeader*)hdr_of(c.ws), loss_rows_all + r0,
        reinterpret_cast<slf_rowstat*>(c.ws + p.off_rowstat) + r0, reinterpret_cast<uint16_t*>(c.ws + p.off_stash),
        reinterpret_cast<uint16_t*>(k.ext_base), (int)(rows - k.ext), rms ? *rms : RmsStep{}));
  }
  if (!dXc && !dW) return SLF_OK;
  ProbSpec ps[2];
  int n = 0;
  SLF_TRY(s_build_bwd(c, a, k, dXc, dx_fp32, dW, ps, &n));
  SchedArena arena;
  if (!sched) {
    const int t = arena.add(ps, n, usable_sms(c.dev) / cta_group());
    SLF_TRY(arena.upload(c));
    sched = arena.dev(c, t);
    sched_stride = arena.tables[t].second;
  }
  return launch_group(c.dev, ps, n, c.s, sched, sched_stride, n == 2 ? SLF_PROF_GEMM_GROUP : -1,
                      in_kernel ? &cj : nullptr);
}

slf_status s_end(Ctx& c, const SArgs& a, int reduction, float scale, float* loss_out, void* dW,
                 const float* rstd = nullptr, const void* gam = nullptr) {
  const Plan& p = c.plan;
  if (dW) {
    ProfScope ps(SLF_PROF_ONEHOT, c.s, 0.0, (double)a.N * a.H * 2 * 2);
    static const bool serial = getenv("SLF_ONEHOT_SERIAL") != nullptr;  // A/B knob: the round-1 kernel
    // segment partials in the tile-partials + stash region (idle after the last chunk): S positions
    // per segment, doubled until [segments][2][H] fp32 fits
    const size_t scratch = p.total - p.off_part;
    int S = 32;
    while ((size_t)((a.N + S - 1) / S) * 8 * a.H > scratch && S < (1 << 30)) S *= 2;
    const unsigned segs = (unsigned)((a.N + S - 1) / S), slabs = (unsigned)((a.H + 1023) / 1024);
    const int32_t* off = reinterpret_cast<const int32_t*>(c.ws + p.off_off);
    const int32_t* idx = reinterpret_cast<const int32_t*>(c.ws + p.off_idx);
    if (serial && !rstd) {
      dim3 grid((unsigned)std::min<int64_t>(a.N, a.V_l), slabs);
      onehot_kernel<<<grid, 128, 0, c.s>>>(reinterpret_cast<const uint16_t*>(a.X), a.H, off, idx,
                                           reinterpret_cast<const int32_t*>(c.ws + p.off_hits), a.V_l, reduction,
                                           scale, 1.0f, hdr_of(c.ws), reinterpret_cast<uint16_t*>(dW));
    } else {
      float* part = reinterpret_cast<float*>(c.ws + p.off_part);
      onehot_seg_kernel<<<dim3(segs, slabs), 128, 0, c.s>>>(reinterpret_cast<const uint16_t*>(a.X), a.H,
                                                             off, reinterpret_cast<const int32_t*>(c.ws + p.off_hits),
                                                             idx, a.V_l, S, reduction, scale, 1.0f, hdr_of(c.ws),
                                                             part, reinterpret_cast<uint16_t*>(dW), rstd,
                                                             reinterpret_cast<const uint16_t*>(gam));
      onehot_join_kernel<<<dim3(segs, slabs), 128, 0, c.s>>>(a.H, off, a.V_l, S, reduction, scale,
                                                              1.0f, hdr_of(c.ws), part,
                                                              reinterpret_cast<uint16_t*>(dW));
    }
    SLF_CUDA(cudaGetLastError());
  }
  if (reduction != SLF_NONE) {
    ProfScope ps(SLF_PROF_LOSS_REDUCE, c.s, 0.0, (double)a.N * 4);
    loss_reduce_kernel<<<1, 1024, 0, c.s>>>(reinterpret_cast<const float*>(c.ws + p.off_loss), a.N, reduction,
                                            hdr_of(c.ws), loss_out);
    SLF_CUDA(cudaGetLastError());
  }
  return SLF_OK;
}

float* s_loss_rows(Ctx& c, int reduction, float* loss_out) {
  return reduction == SLF_NONE ? loss_out : reinterpret_cast<float*>(c.ws + c.plan.off_loss);
}

// Row chunks of the fused single-GPU call.  With `extend` (dhidden requested), a full chunk grows
// by E rows whose stash lives in dhidden's not-yet-written rows beyond it: E*ld_stash <=
// (N - r0 - C - E)*H, a multiple of 256 (no half-empty CTA-pair row tiles; measured 2 % faster
// than 128 despite one more chunk), at most C (partials room).  SLF_S_NO_EXT=1 disables it.
std::vector<SChunk> s_chunks(const Plan& p, int64_t N, int64_t H, bool extend, uint8_t* dX) {
  static const bool no_ext = getenv("SLF_S_NO_EXT") != nullptr;
  static const int64_t ext_gran = getenv("SLF_S_EXT_GRAN") ? atoi(getenv("SLF_S_EXT_GRAN")) : 256;
  static const bool no_pref = getenv("SLF_S_REF_EXT") && atoi(getenv("SLF_S_REF_EXT")) == 0;
  // X'^T [H][rows rounded to 8] fits in dhidden's rows after the chunk and its extended stash: the
  // chunk can take the per-row stash reference (phase_s) instead of the in-place rescale
  auto xt_fits = [&](int64_t r0, int64_t rows, int64_t e) {
    const size_t lo = align_up((size_t)(r0 + rows) * H * 2 + (size_t)e * p.ld_stash * 2, 1024);
    return lo + (size_t)H * ((rows + 7) / 8 * 8) * 2 <= (size_t)N * H * 2;
  };
  // pref: a chunk whose extension would leave no room for X'^T takes the largest extension that
  // does (its rows move to the chunks after it) — kept when a simple cost model says it is cheaper:
  // an extra chunk costs its launch tails (~60 us) plus a W read pass and a dW read-modify-write
  // (8 V H bytes, mostly hidden under the MMAs: counted at 50 TB/s); a chunk on the in-place rescale
  // costs a fully exposed pass over its stash (4 rows V bytes at 5 TB/s) plus its combine launch.
  // Llama-8B: 19 chunks either way, 1 instead of 3 rescaled; Llama-70B: 16 instead of 15 chunks,
  // 2 instead of 13 rescaled.
  auto build = [&](bool pref) {
  std::vector<SChunk> chunks;
  for (int64_t r0 = 0, ci = 0; r0 < N; ++ci) {
    SChunk k{ci, r0, std::min(p.C, N - r0), 0, nullptr, nullptr, 0};
    if (extend && !no_ext && k.rows == p.C) {
      const int64_t free_rows = N - r0 - p.C;
      int64_t e = free_rows > 0 ? (free_rows * H) / (p.ld_stash + H) : 0;
      e = std::min<int64_t>(e, p.C) / ext_gran * ext_gran;
      if (pref && e > 0 && xt_fits(r0, p.C, 0) && !xt_fits(r0, p.C + e, e))
        while (e > 0 && !xt_fits(r0, p.C + e, e)) e -= ext_gran;
      if (e > 0) {
        k.ext = e;
        k.rows = p.C + e;
        k.ext_base = dX ? dX + (size_t)(r0 + k.rows) * H * 2 : nullptr;
      }
    }
    // X_chunk^T after the extended stash in dhidden's unwritten rows, when it fits (SLF_XT=1 only).
    // Off by default: it makes the dW tiles 6 % faster per clock (both operands MN-major cost ~9 %),
    // but under the 1 kW power cap the step was 0.3 ms SLOWER (46.63 +- 0.21 vs 46.32 +- 0.13 ms,
    // five alternating pairs on one box; the transposes add 0.25 ms per step).  DESIGN.md §7b.
    static const bool no_xt = !(getenv("SLF_XT") && atoi(getenv("SLF_XT")) == 1);
    if (extend && dX && !no_xt) {
      const size_t lo = align_up((size_t)(r0 + k.rows) * H * 2 + (size_t)k.ext * p.ld_stash * 2, 1024);
      const int64_t ld = (k.rows + 7) / 8 * 8;
      if (lo + (size_t)H * ld * 2 <= (size_t)N * H * 2) {
        k.xt = dX + lo;
        k.ld_xt = ld;
      }
    }
    chunks.push_back(k);
    r0 += k.rows;
  }
  return chunks;
  };
  std::vector<SChunk> greedy = build(false);
  if (!extend || no_ext || no_pref) return greedy;
  std::vector<SChunk> pref = build(true);
  auto cost = [&](const std::vector<SChunk>& v) {
    const double Vd = (double)p.ld_stash, Hd = (double)H;
    double t = (double)v.size() * (60e-6 + 8.0 * Vd * Hd / 50e12);
    for (const SChunk& k : v)
      if (!xt_fits(k.r0, k.rows, k.ext)) t += 4.0 * (double)k.rows * Vd / 5e12 + 20e-6;
    return t;
  };
  return cost(pref) < cost(greedy) ? pref : greedy;
}

// The fused single-GPU call under schedule S (g = 1: a chunk's statistics are its own).  When dX
// is requested, the chunks are extended into dhidden's not-yet-written rows (s_chunks): fewer
// chunks, fewer dW accumulation passes and longer dW K, at no extra memory.
// The final RMSNorm fused into the chunk loop (slf_rmsnorm_lce_fwd_bwd): X is the
// RMSNorm input x; chunk k's y rows live in ybuf[k & 1].  The RMSNorm jobs of a chunk boundary ride
// in chunk k's combine_transform launch (rmsnorm.cuh RmsStep): dx of chunk k-2, dg partials of
// chunk k-1, y of chunk k+1, the dg sum of chunk k-2; one launch before the loop (y of chunk 0)
// and two after it.
struct RmsFuse {
  const void* g;
  float eps;
  float* dg;          // caller's fp32 [H]
  uint8_t* ybuf[2];   // [max chunk rows][H] bf16, by chunk parity
  float* rstd;        // [N]
  float* part[2];     // [max row groups][H] fp32 dg partials, by chunk parity
  float* mref;        // [N] per-row stash reference (the plan's array)
};

// The RMSNorm jobs of one launch, for chunks (by index; -1 = none): dx of cx, dg partials of cp,
// y of cf, dg sum of cr.
RmsStep rms_jobs(const SArgs& a, const RmsFuse& rf, void* dX, const std::vector<SChunk>& ch, int64_t cx, int64_t cp,
                 int64_t cf, int64_t cr) {
  const int64_t n = (int64_t)ch.size();
  RmsStep r{};
  r.x = reinterpret_cast<const uint16_t*>(a.X);
  r.g = reinterpret_cast<const uint16_t*>(rf.g);
  r.H = a.H;
  r.eps = rf.eps;
  r.rstd = rf.rstd;
  r.dx = reinterpret_cast<uint16_t*>(dX);
  if (cx >= 0 && cx < n) {
    r.x_r0 = ch[cx].r0;
    r.x_rows = ch[cx].rows;
  }
  if (cp >= 0 && cp < n) {
    r.p_r0 = ch[cp].r0;
    r.p_rows = ch[cp].rows;
    r.part_w = rf.part[cp & 1];
  }
  if (cf >= 0 && cf < n) {
    r.f_r0 = ch[cf].r0;
    r.f_rows = ch[cf].rows;
    r.ybuf = reinterpret_cast<uint16_t*>(rf.ybuf[cf & 1]);
    if (ch[cf].ref) {  // the chunk's per-row stash reference from its y rows
      r.W = reinterpret_cast<const uint16_t*>(a.W);
      r.t = a.t;
      r.ignore_index = a.ign;
      r.V = a.V_l;
      r.shift = STASH_REF_SHIFT;
      r.mref = rf.mref;
    }
  }
  if (cr >= 0 && cr < n) {
    r.red_ngroups = (int)((ch[cr].rows + RMS_RG - 1) / RMS_RG);
    r.red_first = cr == 0;
    r.part_r = rf.part[cr & 1];
    r.dg = rf.dg;
  }
  return r;
}

slf_status launch_rms_step(Ctx& c, const RmsStep& r) {
  const int64_t blocks = rms_blocks_of(r);
  if (!blocks) return SLF_OK;
  ProfScope ps(SLF_PROF_RMSNORM, c.s, 0.0,
               (double)(r.x_rows * 3 + r.p_rows * 2 + r.f_rows * 2) * r.H * 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(RMS_THREADS);
  cfg.stream = c.s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SLF_CUDA(cudaLaunchKernelEx(&cfg, rms_step_kernel, r));
  return SLF_OK;
}

slf_status phase_s(Ctx& c, const void* X, const void* W, const int32_t* t, int64_t N, int64_t H, int64_t V,
                   int32_t ignore_index, int reduction, float scale, float* loss_out, void* dX, void* dW,
                   const RmsFuse* rf = nullptr) {
  const Plan& p = c.plan;
  const SArgs a{X, W, t, N, H, V, 0, V, ignore_index};
  SLF_TRY(s_begin(c, a, dW != nullptr));
  std::vector<SChunk> chunks = s_chunks(p, N, H, dX != nullptr, reinterpret_cast<uint8_t*>(dX));
  // Per-row stash reference (SLF_S_CLASSIC=1: the in-place rescale for every chunk).
  // X'_chunk goes over the fused RMSNorm's y buffer, else into dhidden's unwritten rows after the
  // chunk's rows and extended stash when it fits there (the last chunks keep the in-place rescale).
  static const bool classic = getenv("SLF_S_CLASSIC") != nullptr;
  bool any_ref = false;
  if (rf)
    for (auto& k : chunks) {  // the chunk's y rows (dW's B operand too); no X^T variant
      k.xrows = rf->ybuf[k.index & 1];
      k.xt = nullptr;
      k.ref = !classic;
      if (k.ref && dW) k.xs = rf->ybuf[k.index & 1];
      any_ref |= k.ref;
    }
  else if (!classic && dX) {
    // X' is written transposed (X'^T [H][rows rounded to 8]: dW's B operand K-major, one MN-major
    // operand instead of two) unless SLF_XS_T=0
    static const bool xs_t = !(getenv("SLF_XS_T") && atoi(getenv("SLF_XS_T")) == 0);
    for (auto& k : chunks) {
      // the chunk takes the reference where X' fits — with or without dW, so that a dX-only call
      // runs the same numerics chunk by chunk (and returns the same bits) as a dX + dW call
      const size_t lo = align_up((size_t)(k.r0 + k.rows) * H * 2 + (size_t)k.ext * p.ld_stash * 2, 1024);
      const int64_t ld = (k.rows + 7) / 8 * 8;
      const size_t need = xs_t ? (size_t)H * ld * 2 : (size_t)k.rows * H * 2;
      if (lo + need <= (size_t)N * H * 2) {
        k.xt = nullptr;
        k.ref = any_ref = true;
        if (!dW) continue;
        if (xs_t) {
          k.xt = reinterpret_cast<uint8_t*>(dX) + lo;
          k.ld_xt = ld;
        } else {
          k.xs = reinterpret_cast<uint8_t*>(dX) + lo;
        }
      }
    }
  }
  // In-kernel combine (SLF_INKERNEL_COMBINE=0: the separate combine launch): chunks
  // with the per-row reference whose X' is X'^T (or no dW), no RMSNorm jobs.
  static const bool cj_off = getenv("SLF_INKERNEL_COMBINE") && atoi(getenv("SLF_INKERNEL_COMBINE")) == 0;
  c.cj_red = reduction;
  c.cj_scale = scale;
  if (!rf && !cj_off && (V + BN - 1) / BN <= 7000)
    for (auto& k : chunks) k.cj = k.ref && (!dW || k.xt) && k.index < WS_SYNC_SLOTS;
  // M_i = x_i . W[t_i] + shift: for every row at once when the inputs are resident; chunk by chunk,
  // after the chunk's rows arrived, in the host-input call
  auto launch_mref = [&](int64_t r0, int64_t rows) -> slf_status {
    ProfScope ps(SLF_PROF_PREP, c.s, 2.0 * rows * H, (double)rows * H * 4);
    mref_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, c.s>>>(
        reinterpret_cast<const uint16_t*>(X) + (size_t)r0 * H, reinterpret_cast<const uint16_t*>(W), t + r0, rows, H,
        ignore_index, 0, V, reinterpret_cast<float*>(c.ws + p.off_mref) + r0);
    SLF_CUDA(cudaGetLastError());
    return SLF_OK;
  };
  const bool mref_per_chunk = any_ref && !rf && c.chunk_ready;
  if (any_ref && !rf && !mref_per_chunk) SLF_TRY(launch_mref(0, N));
  // LPT tables per distinct chunk shape (rows, ext, first/RMW), uploaded once.
  SchedArena arena;
  std::vector<std::pair<std::pair<int64_t, int64_t>, int>> keys;
  std::vector<int> tab(chunks.size(), -1);
  if (dX || dW) {
    for (size_t i = 0; i < chunks.size(); ++i) {
      const auto key = std::make_pair(chunks[i].rows, chunks[i].ext);
      int found = -1;
      for (auto& kk : keys)
        if (kk.first == key) found = kk.second;
      if (found < 0) {
        ProbSpec ps[2];
        int n = 0;
        SChunk rep = chunks[i];
        rep.index = std::max<int64_t>(rep.index, 1);  // model the common read-modify-write case
        SLF_TRY(s_build_bwd(c, a, rep, dX ? (uint8_t*)dX + (size_t)rep.r0 * H * 2 : nullptr, 0, dW, ps, &n));
        found = arena.add(ps, n, usable_sms(c.dev) / cta_group());
        keys.push_back({key, found});
      }
      tab[i] = found;
    }
    if (arena.fits(c))
      SLF_TRY(arena.upload(c));
    else
      std::fill(tab.begin(), tab.end(), -1);  // too many shapes: each launch uploads its own table
  }
  float* loss_rows = s_loss_rows(c, reduction, loss_out);
  if (c.enqueue_inputs) SLF_TRY(c.enqueue_inputs());
  for (size_t i = 0; i < chunks.size(); ++i) {
    const SChunk& k = chunks[i];
    // Input rows: chunks 0 and 1 wait for their own copies; chunk 2 waits for the last copy (the
    // copy stream is FIFO, so all rows are then present; by then two chunks of GEMMs have hidden
    // the transfer).  Few waits: a stream wait between two kernels forfeits the programmatic
    // dependent launch overlap of the kernel after it.
    if (c.chunk_ready && i <= 2)
      SLF_CUDA(cudaStreamWaitEvent(c.s, c.chunk_ready[i < 2 ? i : chunks.size() - 1], 0));
    if (k.xt && dW && !k.ref) SLF_TRY(launch_transpose_x(c, a, k));
    if (mref_per_chunk && k.ref) SLF_TRY(launch_mref(k.r0, k.rows));
    if (rf && i == 0) SLF_TRY(launch_rms_step(c, rms_jobs(a, *rf, dX, chunks, -1, -1, 0, -1)));  // y of chunk 0
    SLF_TRY(s_chunk_stats(c, a, k, nullptr));
    const int64_t ki = (int64_t)i;
    const RmsStep jobs = rf ? rms_jobs(a, *rf, dX, chunks, ki - 2, ki - 1, ki + 1, ki - 2) : RmsStep{};
    SLF_TRY(s_chunk_bwd(c, a, k, nullptr, 1, reduction, scale, loss_rows,
                        dX ? reinterpret_cast<uint8_t*>(dX) + (size_t)k.r0 * H * 2 : nullptr, 0, dW,
                        tab[i] >= 0 ? arena.dev(c, tab[i]) : nullptr, tab[i] >= 0 ? arena.tables[tab[i]].second : 0,
                        rf ? &jobs : nullptr));
  }
  if (rf) {  // dx of the last two chunks, dg partials of the last, the last two dg sums
    const int64_t n = (int64_t)chunks.size();
    SLF_TRY(launch_rms_step(c, rms_jobs(a, *rf, dX, chunks, n - 2, n - 1, -1, n - 2)));
    SLF_TRY(launch_rms_step(c, rms_jobs(a, *rf, dX, chunks, n - 1, -1, -1, n - 1)));
    return s_end(c, a, reduction, scale, loss_out, dW, rf->rstd, rf->g);
  }
  return s_end(c, a, reduction, scale, loss_out, dW);
}

// Plan selection: SLF_SCHED_S for the fused single-GPU call when it fits (no recompute),
// otherwise schedule R; the split / shard entry points always use R.
bool plan_any(int64_t N, int64_t H, int64_t V, int schedule, size_t budget, bool allow_s, Plan* out) {
  if ((schedule == SLF_SCHED_S || schedule == SLF_SCHED_AUTO) && allow_s && plan_s(N, H, V, budget, out)) return true;
  if (schedule == SLF_SCHED_S) return false;
  return plan_r(N, H, V, budget, out);
}

slf_status setup(Ctx& c, int64_t N, int64_t H, int64_t V_l, size_t budget, void* ws, size_t ws_bytes, void* stream,
                 int schedule = SLF_SCHED_R, bool allow_s = false) {
  SLF_TRY(device_info(&c.dev));
  if (!plan_any(N, H, V_l, schedule, budget, allow_s, &c.plan))
    return fail(SLF_ERR_WORKSPACE, "no plan fits the budget (N=%lld H=%lld V=%lld budget=%zu schedule=%d)",
                (long long)N, (long long)H, (long long)V_l, budget ? budget : default_budget(N, V_l), schedule);
  if (ws_bytes < c.plan.total)
    return fail(SLF_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, c.plan.total);
  c.s = reinterpret_cast<cudaStream_t>(stream);
  c.ws = reinterpret_cast<uint8_t*>(ws);
  return SLF_OK;
}


// ---- vocab-sharded step with in-library collectives (slf_lce_fwd_bwd_sharded) ------
void shard_bounds(int64_t V, int g, int k, int64_t* v0, int64_t* vl) {
  const int64_t a = V * k / g, b = V * (k + 1) / g;
  *v0 = a;
  *vl = b - a;
}

// The rank's workspace: [ schedule-S workspace (planner budget b) | dX partial [2C][H] fp32 |
// local stats 2C*16 | gathered stats g*2C*16 ], b the largest planner budget whose total fits.
// Chunks are extended into dhidden's unwritten rows as in the fused call (up to 2C rows), so the
// partial and the statistics buffers hold 2C rows; the partial is single-buffered (the chunk's dX
// all-reduce shares the communicator stream with the next chunk's statistics all-gather, so it is
// complete by the time the next chunk's combine runs anyway).
struct ShardPlan {
  Plan p;
  size_t b, off_dx, off_st, off_all, total;
  int64_t v0, V_l;
  // The fp32 dX partial: with ws_part a dedicated [2C][H] workspace region (round 1
  // layout); otherwise at the top of dhidden's unwritten rows, and for the last chunks (whose rows
  // leave no room there) in the tail of the workspace stash, those chunks being r_tail rows.
  bool ws_part = true;
  int64_t r_tail = 0;
  bool xt_tail = false;  // tail chunks hold X'^T after their partial (per-row stash reference)
};

// Stash row pitches of the largest / smallest shard (every rank cuts the same chunks from these).
int64_t shard_ld_max(int64_t Vg, int g) { return (int64_t)align_up((size_t)((Vg + g - 1) / g), 8); }
int64_t shard_ld_min(int64_t Vg, int g) { return (int64_t)align_up((size_t)(Vg / g), 8); }

// Rows of a chunk whose stash, fp32 partial and X'^T share the workspace stash of C rows on EVERY
// rank: R * ld_max * 2 (rounded to 1 KB) + R * H * 4 (rounded) + H * R * 2 <= C * ld_min * 2; a
// multiple of 8 (X'^T pitch).
// Also X'^T [H][R] after the partial (the per-row stash reference, for tail chunks).
size_t shard_tail_bytes(int64_t R, int64_t H, int64_t ld_max, bool xt) {
  const size_t sp = align_up((size_t)R * ld_max * 2, 1024) + (size_t)R * H * 4;
  return xt ? align_up(sp, 1024) + (size_t)H * R * 2 : sp;
}
int64_t shard_tail_rows(int64_t C, int64_t H, int64_t ld_max, int64_t ld_min, bool xt) {
  const double cap = (double)C * ld_min * 2 - 2048;
  int64_t R = (int64_t)(cap / ((double)ld_max * 2 + (double)H * (xt ? 6 : 4))) / 8 * 8;
  while (R > 0 && shard_tail_bytes(R, H, ld_max, xt) > (size_t)C * ld_min * 2) R -= 8;
  return std::max<int64_t>(R, 0);
}

// mode 0: the partial in a workspace region; 1: at dhidden's top (tail chunks: workspace stash
// tail); 2: as 1, with room for the tail chunks' X'^T too
bool shard_layout(int64_t N, int64_t H, int64_t V_l, int64_t Vg, int g, int mode, size_t b, ShardPlan* sp) {
  const bool top = mode != 0;
  if (!plan_s(N, H, V_l, b, &sp->p)) return false;
  const int64_t C2 = 2 * sp->p.C;
  const int64_t ldx = shard_ld_max(Vg, g), ldn = shard_ld_min(Vg, g);
  // top: the partial leaves the workspace (shard_plan picks the layout with fewer chunks)
  sp->ws_part = !top;
  sp->xt_tail = mode == 2;
  sp->r_tail = sp->ws_part ? 0 : shard_tail_rows(sp->p.C, H, ldx, ldn, sp->xt_tail);
  if (!sp->ws_part && sp->r_tail < 8) return false;
  sp->b = b;
  sp->off_dx = align_up(sp->p.total, 1024);
  sp->off_st = align_up(sp->off_dx + (sp->ws_part ? (size_t)C2 * H * 4 : 0), 1024);
  sp->off_all = align_up(sp->off_st + (size_t)C2 * 16, 1024);
  sp->total = sp->off_all + (size_t)g * C2 * 16;
  return true;
}

// The chunks every rank cuts (identical on all ranks: every size below is computed from the largest
// shard's stash row pitch ld_max) and where each chunk's fp32 dX partial P lives.
// With a dhidden (dX) and !ws_part, chunk c's partial goes to the top of dhidden, [D - rows*H*4, D)
// with D = N*H*2, while it fits above the chunk's own rows, its extended stash and its X'^T (X'^T
// must not overlap the partial its group writes); the previous chunk's partial is still in flight
// (its all-reduce / P2P reads overlap this chunk's stash GEMM), so this chunk's extended stash also
// stays below that one.  From the first chunk that does not fit on, chunks are r_tail rows (no
// extension) and P sits in the workspace stash after the chunk's rows (the next chunk's stash GEMM
// writes only the first r_tail rows, so it never touches the partial in flight).  X'^T (written by
// the chunk's combine, after the previous chunk's partial was reduced and read) only has to stay
// below the chunk's own partial.
std::vector<SChunk> shard_chunks(const ShardPlan& sp, int64_t N, int64_t H, int64_t Vg, int g, bool extend,
                                 uint8_t* dX) {
  Plan pe = sp.p;
  pe.ld_stash = shard_ld_max(Vg, g);
  if (!extend || sp.ws_part) {
    std::vector<SChunk> v = s_chunks(pe, N, H, extend, dX);
    for (SChunk& k : v) {
      k.part_off = PART_WS_REGION;
      k.xt_lim = (size_t)N * H * 2;
    }
    return v;
  }
  static const bool no_ext = getenv("SLF_S_NO_EXT") != nullptr;
  static const int64_t ext_gran = getenv("SLF_S_EXT_GRAN") ? atoi(getenv("SLF_S_EXT_GRAN")) : 256;
  static const bool no_pref = getenv("SLF_S_REF_EXT") && atoi(getenv("SLF_S_REF_EXT")) == 0;
  const int64_t C = pe.C, ld = pe.ld_stash;
  const size_t D = (size_t)N * H * 2;
  // X'^T [H][rows rounded to 8] fits between the chunk's extended stash and its partial
  // (phase_sharded's per-row-reference rule for a top chunk)
  auto xt_ok = [&](int64_t r0, int64_t rows, int64_t e) {
    const size_t lo = align_up((size_t)(r0 + rows) * H * 2 + (size_t)e * ld * 2, 1024);
    return lo + (size_t)H * ((rows + 7) / 8 * 8) * 2 <= D - (size_t)rows * H * 4;
  };
  // pref: as s_chunks — a top chunk takes the largest extension (or, without one, the longest
  // shorter length) that leaves room for X'^T when one does; the plan is kept if the cost model
  // prefers it
  auto build = [&](bool pref) {
  std::vector<SChunk> chunks;
  size_t prev_q = 0;  // bytes at dhidden's top held by the previous chunk's partial
  bool tail = false;
  int64_t tail_rows = 0;
  for (int64_t r0 = 0, ci = 0; r0 < N; ++ci) {
    SChunk k{ci, r0, 0, 0, nullptr, nullptr, 0};
    const int64_t base = std::min(C, N - r0);
    if (!tail) {
      int64_t e0 = 0;
      if (!no_ext && base == C) {
        const int64_t free_rows = N - r0 - C;
        e0 = free_rows > 0 ? std::min<int64_t>((free_rows * H) / (ld + H), C) / ext_gran * ext_gran : 0;
      }
      bool ok = false;
      for (int pass = pref ? 0 : 1; pass < 2 && !ok; ++pass) {  // pass 0: only extensions with room for X'^T
        for (int64_t e = e0; e >= 0; e -= ext_gran) {
          const int64_t rows = base + e;
          const size_t end = (size_t)(r0 + rows) * H * 2;  // the chunk's own rows end here
          if (end + (size_t)rows * H * 4 > D) continue;
          // the extended stash is written while the previous partial is in flight and read while
          // this chunk's partial is written
          if (e > 0 && end + (size_t)e * ld * 2 > D - std::max(prev_q, (size_t)rows * H * 4)) continue;
          if (pass == 0 && !xt_ok(r0, rows, e)) continue;
          ok = true;
          k.rows = rows;
          k.ext = e;
          break;
        }
      }
      if (pref && ok && k.ext == 0 && !xt_ok(r0, k.rows, 0)) {  // a shorter chunk with room for X'^T
        const int64_t r = (N - r0) / 4 / 256 * 256;
        if (r >= 256 && r > sp.r_tail && xt_ok(r0, r, 0)) k.rows = r;
      }
      if (!ok) {  // a shorter chunk (no extension) whose partial still fits above its rows
        const int64_t r = (N - r0) / 3 / 256 * 256;
        if (r > sp.r_tail) {
          ok = true;
          k.rows = r;
          k.ext = 0;
        }
      }
      if (ok) {
        k.part_off = (int64_t)(D - (size_t)k.rows * H * 4);
        k.xt_lim = (size_t)k.part_off;  // X'^T is written after the previous partial was consumed
        if (k.ext) k.ext_base = dX ? dX + (size_t)(r0 + k.rows) * H * 2 : nullptr;
        prev_q = (size_t)k.rows * H * 4;
      } else {
        tail = true;
        // whole 256-row tiles where the tail allows them (a 696-row chunk computes 768 rows'
        // worth of stash and dX tiles), else an even split
        const int64_t M = N - r0, R256 = sp.r_tail / 256 * 256;
        if (R256 >= 256) {
          tail_rows = R256;
        } else {
          const int64_t n = (M + sp.r_tail - 1) / sp.r_tail;
          tail_rows = std::min<int64_t>(sp.r_tail, ((M + n - 1) / n + 7) / 8 * 8);
        }
      }
    }
    if (tail) {
      k.rows = std::min(tail_rows, N - r0);
      k.part_off = PART_WS_TAIL;
      k.xt_lim = D;
    }
    chunks.push_back(k);
    r0 += k.rows;
  }
  return chunks;
  };
  std::vector<SChunk> greedy = build(false);
  if (no_pref) return greedy;
  std::vector<SChunk> pref = build(true);
  auto cost = [&](const std::vector<SChunk>& v) {  // the model of s_chunks
    double t = (double)v.size() * (60e-6 + 8.0 * (double)ld * (double)H / 50e12);
    for (const SChunk& k : v) {
      const bool ref = k.part_off == PART_WS_TAIL ? sp.xt_tail : xt_ok(k.r0, k.rows, k.ext);
      if (!ref) t += 4.0 * (double)k.rows * (double)ld / 5e12 + 20e-6;
    }
    return t;
  };
  return cost(pref) < cost(greedy) ? pref : greedy;
}

// The largest planner budget whose layout fits `total` with a row chunk of at most c_cap (0: any).
bool shard_fit(int64_t N, int64_t H, int64_t V_l, int64_t Vg, int g, int mode, size_t total, int64_t c_cap,
               ShardPlan* sp) {
  auto ok = [&](size_t b) {
    return shard_layout(N, H, V_l, Vg, g, mode, b, sp) && sp->total <= total && (c_cap == 0 || sp->p.C <= c_cap);
  };
  // bisection (the layout grows with the budget; 0 would mean the default): below the smallest
  // feasible planner budget the predicate counts as "go larger", so it is monotone
  auto below_or_ok = [&](size_t b) { return !shard_layout(N, H, V_l, Vg, g, mode, b, sp) || ok(b); };
  size_t lo = 1, hi = total;
  while (lo < hi) {
    const size_t mid = lo + (hi - lo + 1) / 2;
    if (below_or_ok(mid))
      lo = mid;
    else
      hi = mid - 1;
  }
  return ok(lo);
}

// Every rank must cut the same row chunks (the statistics are exchanged chunk by chunk), but shard
// sizes differ by one row when g does not divide V: the chunk C is the one the LARGEST shard
// (ceil(V/g) rows) fits, and each rank takes the largest planner budget giving exactly that C.
bool shard_plan(int64_t N, int64_t H, int64_t Vg, int g, int k, size_t budget, ShardPlan* out) {
  if (N < 1 || H < 8 || Vg < 1 || g < 1 || k < 0 || k >= g || Vg < g) return false;
  int64_t v0, vl;
  shard_bounds(Vg, g, k, &v0, &vl);
  const size_t total = budget ? budget : default_budget(N, Vg);
  // The placements of the fp32 dX partial (shard_layout modes 2, 1, 0); the one cutting fewer row
  // chunks wins, then the one leaving fewer chunks on the in-place rescale (ties: the earlier mode).
  // Everything here is the same on every rank.
  ShardPlan best;
  size_t best_n = 0;
  int best_cl = 0;
  static const char* force = getenv("SLF_SHARD_PART");  // "top" / "region": one placement only (tests)
  const int64_t ldx = shard_ld_max(Vg, g);
  for (const int mode : {2, 1, 0}) {
    if (force && strcmp(force, mode ? "region" : "top") == 0) continue;
    ShardPlan big, sp;
    if (!shard_fit(N, H, (Vg + g - 1) / g, Vg, g, mode, total, 0, &big)) continue;
    if (!shard_fit(N, H, vl, Vg, g, mode, total, big.p.C, &sp) || sp.p.C != big.p.C) continue;
    ShardPlan small;  // the same decision on every rank: the smallest shard must fit this C too
    if (!shard_fit(N, H, Vg / g, Vg, g, mode, total, big.p.C, &small) || small.p.C != big.p.C) continue;
    sp.v0 = v0;
    sp.V_l = vl;
    const std::vector<SChunk> ch = shard_chunks(sp, N, H, Vg, g, true, nullptr);
    int cl = 0;  // chunks without room for X'^T (phase_sharded's rule)
    for (const SChunk& k : ch) {
      if (k.part_off == PART_WS_TAIL && sp.xt_tail) continue;
      const size_t lo = align_up((size_t)(k.r0 + k.rows) * H * 2 + (size_t)k.ext * ldx * 2, 1024);
      cl += lo + (size_t)H * ((k.rows + 7) / 8 * 8) * 2 > k.xt_lim;
    }
    if (best_n == 0 || ch.size() < best_n || (ch.size() == best_n && cl < best_cl)) {
      best = sp;
      best_n = ch.size();
      best_cl = cl;
    }
  }
  if (best_n == 0) return false;
  *out = best;
  return true;
}

slf_status comm_fail_nccl(ncclResult_t r, const char* what) {
  NcclApi& api = nccl_api();
  return fail(SLF_ERR_COMM, "%s: %s", what, api.GetErrorString ? api.GetErrorString(r) : "nccl error");
}

// All-gather of `bytes` per rank, the result visible to later work on s.
slf_status comm_allgather(slf_comm cm, const void* send, void* recv, size_t bytes, cudaStream_t s) {
  if (cm->world == 1) {
    if (recv != send) SLF_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
    if (!cm->nccl && !cm->cb_allgather) return SLF_OK;
  }
  if (cm->cb_allgather) {
    if (cm->cb_allgather(send, recv, bytes, s, cm->cb_user) != 0) return fail(SLF_ERR_COMM, "allgather callback failed");
    return SLF_OK;
  }
  NcclApi& api = nccl_api();
  SLF_CUDA(cudaEventRecord(cm->ev_in, s));
  SLF_CUDA(cudaStreamWaitEvent(cm->cs, cm->ev_in, 0));
  ncclResult_t r;
  {
    ProfScope ps(SLF_PROF_COMM_ALLGATHER, cm->cs, 0.0, (double)bytes * cm->world);
    r = api.AllGather(send, recv, bytes, ncclUint8, cm->nccl, cm->cs);
  }
  if (r != ncclSuccess) return comm_fail_nccl(r, "ncclAllGather");
  SLF_CUDA(cudaEventRecord(cm->ev_ag, cm->cs));
  SLF_CUDA(cudaStreamWaitEvent(s, cm->ev_ag, 0));
  return SLF_OK;
}

// In-place fp32 sum all-reduce of buf[count], started after the work on s so far; completion is
// joined to s by comm_join(slot).
slf_status comm_allreduce_start(slf_comm cm, float* buf, size_t count, int slot, cudaStream_t s) {
  if (cm->cb_allreduce) {
    if (cm->cb_allreduce(buf, count, s, cm->cb_user) != 0) return fail(SLF_ERR_COMM, "allreduce callback failed");
    return SLF_OK;
  }
  if (!cm->nccl) return SLF_OK;  // world 1 without a transport: the partial is the sum
  NcclApi& api = nccl_api();
  SLF_CUDA(cudaEventRecord(cm->ev_in, s));
  SLF_CUDA(cudaStreamWaitEvent(cm->cs, cm->ev_in, 0));
  ncclResult_t r;
  {
    ProfScope ps(SLF_PROF_COMM_ALLREDUCE, cm->cs, 0.0, (double)count * 4);
    r = api.AllReduce(buf, buf, count, ncclFloat32, ncclSum, cm->nccl, cm->cs);
  }
  if (r != ncclSuccess) return comm_fail_nccl(r, "ncclAllReduce");
  SLF_CUDA(cudaEventRecord(cm->ev_ar[slot], cm->cs));
  return SLF_OK;
}

slf_status comm_join(slf_comm cm, int slot, cudaStream_t s) {
  if (cm->nccl && !cm->cb_allreduce) SLF_CUDA(cudaStreamWaitEvent(s, cm->ev_ar[slot], 0));
  return SLF_OK;
}

// ---- data-parallel (token-sharded) step with in-library collectives (slf_lce_fwd_bwd_dp) --------
// The MEAN denominator must be the GLOBAL valid count: right after the target scan the header's
// n_valid is summed across ranks on the device (no host round trip), so every later kernel (coef,
// loss) sees the global count.  Float transports carry it as three 16-bit limbs (exact for any
// count < 2^48 and up to 256 ranks).
__global__ void u64_to_limbs_kernel(const unsigned long long* n, float* limbs) {
  const unsigned long long v = *n;
  limbs[0] = (float)(v & 0xffffull);
  limbs[1] = (float)((v >> 16) & 0xffffull);
  limbs[2] = (float)((v >> 32) & 0xffffull);
}
__global__ void limbs_to_u64_kernel(const float* limbs, unsigned long long* n) {
  *n = (unsigned long long)limbs[0] + ((unsigned long long)limbs[1] << 16) + ((unsigned long long)limbs[2] << 32);
}

slf_status comm_allreduce_now(slf_comm cm, float* buf, size_t count, cudaStream_t s) {
  SLF_TRY(comm_allreduce_start(cm, buf, count, 0, s));
  return comm_join(cm, 0, s);
}


void p2p_release(slf_comm cm) {
  for (auto& kv : cm->ipc_open) cudaIpcCloseMemHandle(kv.second);
  cm->ipc_open.clear();
  cm->dx_epoch = 0;
  for (int r = 0; r < cm->world && r < P2P_MAX_RANKS; ++r)
    if (cm->p2p_peer[r] && r != cm->rank) cudaIpcCloseMemHandle(cm->p2p_peer[r]);
  if (cm->p2p_buf) cudaFree(cm->p2p_buf);
  cm->p2p_buf = nullptr;
  memset(cm->p2p_peer, 0, sizeof(cm->p2p_peer));
  cm->p2p_rows = 0;
  cm->epoch = 0;
}

size_t p2p_data_off(const slf_comm_s* cm, unsigned long long epoch) {
  return P2P_HDR_BYTES + (size_t)(epoch & 1) * cm->world * cm->p2p_rows * 16;
}

// (Re)allocate this rank's receive buffer for `rows` rows per slot and map every peer's (a
// collective: every rank reaches it at the same call, their chunk plans being identical).
slf_status p2p_ensure(slf_comm cm, int64_t rows, cudaStream_t s) {
  if (cm->p2p_buf && cm->p2p_rows >= rows) return SLF_OK;
  if (cm->world > P2P_MAX_RANKS) return fail(SLF_ERR_ARG, "P2P statistics exchange supports <= %d ranks", P2P_MAX_RANKS);
  SLF_CUDA(cudaStreamSynchronize(s));
  p2p_release(cm);
  cm->p2p_rows = rows;
  const size_t bytes = P2P_HDR_BYTES + 2 * (size_t)cm->world * rows * 16;
  if (!cm->p2p_err_host) {  // sticky timeout flag readable by the host without a synchronisation
    SLF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&cm->p2p_err_host), 64, cudaHostAllocMapped));
    *cm->p2p_err_host = 0;
    SLF_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&cm->p2p_err_dev), cm->p2p_err_host, 0));
  }
  SLF_CUDA(cudaMalloc(&cm->p2p_buf, bytes));
  SLF_CUDA(cudaMemset(cm->p2p_buf, 0, bytes));
  SLF_CUDA(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  SLF_CUDA(cudaIpcGetMemHandle(&h, cm->p2p_buf));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  uint8_t* dev = nullptr;  // the handles travel through the communicator's own all-gather
  SLF_CUDA(cudaMalloc(&dev, 64 * (size_t)(cm->world + 1)));
  std::vector<uint8_t> all((size_t)64 * cm->world);
  slf_status st = SLF_OK;
  if (cudaMemcpy(dev, &h, 64, cudaMemcpyHostToDevice) != cudaSuccess)
    st = fail(SLF_ERR_CUDA, "handle upload failed");
  if (st == SLF_OK) st = comm_allgather(cm, dev, dev + 64, 64, s);
  if (st == SLF_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(SLF_ERR_CUDA, "handle exchange failed");
  if (st == SLF_OK && cudaMemcpy(all.data(), dev + 64, all.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
    st = fail(SLF_ERR_CUDA, "handle download failed");
  cudaFree(dev);
  for (int r = 0; st == SLF_OK && r < cm->world; ++r) {
    if (r == cm->rank) {
      cm->p2p_peer[r] = cm->p2p_buf;
      continue;
    }
    cudaIpcMemHandle_t ph;
    memcpy(&ph, all.data() + (size_t)64 * r, 64);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, ph, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) st = fail(SLF_ERR_COMM, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
    cm->p2p_peer[r] = static_cast<uint8_t*>(p);
  }
  if (st != SLF_OK) {
    p2p_release(cm);
    return st;
  }
  // every rank has mapped every buffer before anyone pushes into one
  float* bar = nullptr;
  SLF_CUDA(cudaMalloc(&bar, 16));
  SLF_CUDA(cudaMemset(bar, 0, 16));
  st = comm_allreduce_start(cm, bar, 4, 0, s);
  if (st == SLF_OK) st = comm_join(cm, 0, s);
  if (st == SLF_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(SLF_ERR_CUDA, "barrier failed");
  cudaFree(bar);
  return st;
}

// One-shot all-gather of this chunk's statistics into every rank's buffer; returns (in *gathered)
// the local [g][rows] view of this epoch.
slf_status p2p_allgather_stats(slf_comm cm, const slf_shardstat* st, int64_t rows, cudaStream_t s,
                               const slf_shardstat** gathered) {
  const unsigned long long e = ++cm->epoch;
  PeerPtrs pp{};
  for (int r = 0; r < cm->world; ++r) pp.p[r] = cm->p2p_peer[r];
  const size_t off = p2p_data_off(cm, e);
  p2p_stats_push_kernel<<<cm->world, 256, 0, s>>>(reinterpret_cast<const uint4*>(st), (int)rows, cm->rank, pp, off);
  SLF_CUDA(cudaGetLastError());
  p2p_stats_wait_kernel<<<1, 32, 0, s>>>(cm->p2p_buf, cm->world, e);
  SLF_CUDA(cudaGetLastError());
  *gathered = reinterpret_cast<const slf_shardstat*>(cm->p2p_buf + off);
  return SLF_OK;
}

typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_memGetAddressRange addr_range_fn() {
  static PFN_memGetAddressRange fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_memGetAddressRange>(p);
  });
  return fn;
}

// Every rank's address of a caller-owned device buffer (e.g. the workspace, dhidden): the
// allocation base is exported by CUDA IPC with the offset inside it, the records are all-gathered
// through the transport, and peers' bases are opened once per handle (cached on the communicator).
slf_status p2p_map(slf_comm cm, const void* local, cudaStream_t s, uint8_t** peer) {
  auto fn = addr_range_fn();
  if (!fn) return fail(SLF_ERR_COMM, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(local)) != CUDA_SUCCESS)
    return fail(SLF_ERR_COMM, "cuMemGetAddressRange failed for %p", local);
  struct Rec {
    cudaIpcMemHandle_t h;
    uint64_t off, pad;
  } rec;
  static_assert(sizeof(Rec) == 80, "80-byte record");
  memset(&rec, 0, sizeof(rec));
  SLF_CUDA(cudaIpcGetMemHandle(&rec.h, reinterpret_cast<void*>(base)));
  rec.off = reinterpret_cast<uint64_t>(local) - (uint64_t)base;
  uint8_t* dev = nullptr;
  SLF_CUDA(cudaMalloc(&dev, sizeof(Rec) * (size_t)(cm->world + 1)));
  std::vector<Rec> all((size_t)cm->world);
  slf_status st = SLF_OK;
  if (cudaMemcpy(dev, &rec, sizeof(Rec), cudaMemcpyHostToDevice) != cudaSuccess) st = fail(SLF_ERR_CUDA, "upload");
  if (st == SLF_OK) st = comm_allgather(cm, dev, dev + sizeof(Rec), sizeof(Rec), s);
  if (st == SLF_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(SLF_ERR_CUDA, "exchange");
  if (st == SLF_OK && cudaMemcpy(all.data(), dev + sizeof(Rec), sizeof(Rec) * all.size(), cudaMemcpyDeviceToHost) !=
                          cudaSuccess)
    st = fail(SLF_ERR_CUDA, "download");
  cudaFree(dev);
  for (int r = 0; st == SLF_OK && r < cm->world; ++r) {
    if (r == cm->rank) {
      peer[r] = static_cast<uint8_t*>(const_cast<void*>(local));
      continue;
    }
    const std::string key(reinterpret_cast<const char*>(&all[r].h), sizeof(cudaIpcMemHandle_t));
    uint8_t* b = nullptr;
    for (auto& kv : cm->ipc_open)
      if (kv.first == key) b = kv.second;
    if (!b) {
      void* p = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&p, all[r].h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return fail(SLF_ERR_COMM, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
      b = static_cast<uint8_t*>(p);
      cm->ipc_open.emplace_back(key, b);
    }
    peer[r] = b + all[r].off;
  }
  return st;
}

// Wait (on stream s) until every rank's counter at `off` in this rank's buffer reached `target`.
slf_status p2p_wait(slf_comm cm, int off, unsigned long long target, cudaStream_t s) {
  p2p_stats_wait_kernel<<<1, 32, 0, s>>>(cm->p2p_buf, cm->world, target, off);
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

slf_status dx_finalize_rows(Ctx& c, const float* dx32, const slf_rowstat* rs, void* out, int64_t rows, int64_t H) {
  const int64_t groups = rows * H / 8;
  const int blocks = (int)std::min<int64_t>((groups + 255) / 256, (int64_t)c.dev->sms * 8);
  ProfScope ps(SLF_PROF_DX_FINALIZE, c.s, 0.0, (double)rows * H * 6 + rows * 16.0);
  dx_finalize_kernel<<<blocks, 256, 0, c.s>>>(dx32, rs, reinterpret_cast<uint16_t*>(out), rows, H);
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

// Per chunk: stash GEMM + local stats -> all-gather -> merge/transform + grouped dX-partial/dW
// launch -> async fp32 all-reduce of the chunk's dX (double-buffered; joined two chunks later, so
// it overlaps the next chunk's stash GEMM) -> bf16 rows.  Mirrors sharded.VocabShardedLCE (S).
slf_status phase_sharded(Ctx& c, const ShardPlan& sp, slf_comm cm, const void* X, const void* W, const int32_t* t,
                         int64_t N, int64_t H, int64_t Vg, int32_t ign, int reduction, float scale, float* loss_out,
                         void* dX, void* dW) {
  const Plan& p = c.plan;
  const int g = cm->world;
  const SArgs a{X, W, t, N, H, sp.V_l, sp.v0, Vg, ign};
  // where a chunk's fp32 dX partial lives (shard_chunks): the workspace region (ws_part), the tail
  // of the workspace stash after r_tail rows, or dhidden's top rows
  const size_t tail_off = p.off_stash + align_up((size_t)sp.r_tail * shard_ld_max(Vg, g) * 2, 1024);
  auto part_of = [&](const SChunk& k) -> float* {
    if (k.part_off == PART_WS_REGION) return reinterpret_cast<float*>(c.ws + sp.off_dx);
    if (k.part_off == PART_WS_TAIL) return reinterpret_cast<float*>(c.ws + tail_off);
    return reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(dX) + k.part_off);
  };
  slf_shardstat* st = reinterpret_cast<slf_shardstat*>(c.ws + sp.off_st);
  slf_shardstat* st_all = reinterpret_cast<slf_shardstat*>(c.ws + sp.off_all);
  const slf_rowstat* rs = reinterpret_cast<const slf_rowstat*>(c.ws + p.off_rowstat);
  const bool p2p_dx = cm->p2p && (cm->p2p_mode & 2) && dX;
  if (cm->p2p) SLF_TRY(p2p_ensure(cm, 2 * p.C, c.s));
  // Peers' fp32 partial buffers are exported themselves (base + offset inside the caller's
  // allocation), not as this rank's workspace offsets: shard sizes differ by one vocabulary row when
  // g does not divide V, and the schedule-S layout (stash leading dimension, CSR arrays) before the
  // partials then differs between ranks.
  uint8_t* part_peer[P2P_MAX_RANKS] = {};
  uint8_t* dx_peer[P2P_MAX_RANKS] = {};
  if (p2p_dx) {  // the same maps on every rank (ws_part is a property of the problem)
    SLF_TRY(p2p_map(cm, c.ws + (sp.ws_part ? sp.off_dx : tail_off), c.s, part_peer));
    SLF_TRY(p2p_map(cm, dX, c.s, dx_peer));
  }
  SLF_TRY(s_begin(c, a, dW != nullptr));
  // Extended chunks (as the fused call): the same on every rank.
  std::vector<SChunk> chunks = shard_chunks(sp, N, H, Vg, g, dX != nullptr, reinterpret_cast<uint8_t*>(dX));
  std::vector<unsigned long long> dx_ep(chunks.size(), 0);
  const int64_t ld_max = (int64_t)align_up((size_t)((Vg + g - 1) / g), 8);
  // Per-row stash reference where X'^T fits in dhidden's rows after the chunk and
  // its extended stash (not finalised yet); M_i needs the global target logit: each shard's
  // contribution, one all-reduce.
  static const bool classic = getenv("SLF_S_CLASSIC") != nullptr;
  bool any_ref = false;
  if (!classic && dX) {
    // tail chunks: X'^T in the workspace stash's tail, after the partial (shard_tail_bytes)
    const size_t xt_tail = align_up(tail_off + (size_t)sp.r_tail * H * 4, 1024);
    for (auto& k : chunks) {
      const int64_t ld = (k.rows + 7) / 8 * 8;
      if (k.part_off == PART_WS_TAIL && sp.xt_tail) {
        k.ref = any_ref = true;
        if (dW) {
          k.xt = c.ws + xt_tail;
          k.ld_xt = ld;
        }
        continue;
      }
      const size_t lo = align_up((size_t)(k.r0 + k.rows) * H * 2 + (size_t)k.ext * ld_max * 2, 1024);
      if (lo + (size_t)H * ld * 2 <= k.xt_lim) {
        k.ref = any_ref = true;
        if (dW) {
          k.xt = reinterpret_cast<uint8_t*>(dX) + lo;
          k.ld_xt = ld;
        }
      }
    }
  }
  // World size 1 (no statistics exchange): the combine runs inside the group launch as in the fused
  // call
  if (g == 1 && !(getenv("SLF_INKERNEL_COMBINE") && atoi(getenv("SLF_INKERNEL_COMBINE")) == 0) &&
      (sp.V_l + BN - 1) / BN <= 7000) {
    c.cj_red = reduction;
    c.cj_scale = scale;
    for (auto& k : chunks) k.cj = k.ref && (!dW || k.xt) && k.index < WS_SYNC_SLOTS;
  }
  if (any_ref) {
    float* mref = reinterpret_cast<float*>(c.ws + p.off_mref);
    {
      ProfScope ps(SLF_PROF_PREP, c.s, 2.0 * N * H, (double)N * H * 4);
      mref_kernel<<<(unsigned)((N * 32 + 255) / 256), 256, 0, c.s>>>(
          reinterpret_cast<const uint16_t*>(X), reinterpret_cast<const uint16_t*>(W), t, N, H, ign, sp.v0, sp.V_l,
          mref, 1);
      SLF_CUDA(cudaGetLastError());
    }
    SLF_TRY(comm_allreduce_now(cm, mref, (size_t)N, c.s));
    mref_finish_kernel<<<(unsigned)((N + 255) / 256), 256, 0, c.s>>>(t, N, ign, Vg, mref);
    SLF_CUDA(cudaGetLastError());
  }
  // LPT tables per distinct chunk shape (rows, ext), uploaded once per call
  SchedArena arena;
  std::vector<std::pair<std::pair<int64_t, int64_t>, int>> keys;
  std::vector<int> tab(chunks.size(), -1);
  if (dX || dW) {
    for (size_t i = 0; i < chunks.size(); ++i) {
      const auto key = std::make_pair(chunks[i].rows, chunks[i].ext);
      int found = -1;
      for (auto& kk : keys)
        if (kk.first == key) found = kk.second;
      if (found < 0) {
        SChunk rep = chunks[i];
        rep.index = std::max<int64_t>(rep.index, 1);
        ProbSpec ps[2];
        int n = 0;
        SLF_TRY(s_build_bwd(c, a, rep, dX ? part_of(chunks[i]) : nullptr, 1, dW, ps, &n));
        found = arena.add(ps, n, usable_sms(c.dev) / cta_group());
        keys.push_back({key, found});
      }
      tab[i] = found;
    }
    if (arena.fits(c))
      SLF_TRY(arena.upload(c));
    else
      std::fill(tab.begin(), tab.end(), -1);
  }
  float* loss_rows = s_loss_rows(c, reduction, loss_out);
  int64_t pending = -1;  // the chunk whose dX all-reduce is in flight (NCCL / callback path)
  auto finish = [&]() -> slf_status {
    const SChunk& k = chunks[pending];
    SLF_TRY(comm_join(cm, 0, c.s));
    SLF_TRY(dx_finalize_rows(c, part_of(k), rs + k.r0, reinterpret_cast<uint8_t*>(dX) + (size_t)k.r0 * H * 2, k.rows, H));
    pending = -1;
    return SLF_OK;
  };
  for (size_t i = 0; i < chunks.size(); ++i) {
    const SChunk& k = chunks[i];
    // World size 1: no statistics to exchange — the merge reads the stash GEMM's tile partials
    // directly, as in the fused call (no shard-statistics pass, no all-gather).  The dX partial
    // and its all-reduce stay (the transport's path).
    const bool solo = g == 1;
    SLF_TRY(s_chunk_stats(c, a, k, solo ? nullptr : st));
    const slf_shardstat* gathered = solo ? nullptr : st_all;
    if (solo) {
    } else if (cm->p2p && (cm->p2p_mode & 1)) {
      SLF_TRY(p2p_allgather_stats(cm, st, k.rows, c.s, &gathered));
    } else {
      SLF_TRY(comm_allgather(cm, st, st_all, (size_t)k.rows * 16, c.s));
    }
    // the previous chunk's all-reduce is complete and its rows are written before this chunk's
    // group rewrites the partial
    if (pending >= 0) SLF_TRY(finish());
    // P2P dX: the partial is rewritten only once every rank has read it (the exchange kernels of
    // chunk i-1 have all signalled)
    if (p2p_dx && i >= 1) SLF_TRY(p2p_wait(cm, (int)P2P_DX_DONE_OFF, dx_ep[i - 1], c.s));
    const int tb = tab[i];
    float* dxp = dX ? part_of(k) : nullptr;
    SLF_TRY(s_chunk_bwd(c, a, k, gathered, g, reduction, scale, loss_rows, dxp, 1, dW,
                        tb >= 0 ? arena.dev(c, tb) : nullptr, tb >= 0 ? arena.tables[tb].second : 0));
    if (p2p_dx) {  // reduce-scatter + all-gather + bf16 finalize of this chunk, one kernel on the comm stream
      dx_ep[i] = ++cm->dx_epoch;
      DxArgs xa{};
      for (int r = 0; r < g; ++r) {
        xa.part.p[r] = k.part_off >= 0 ? dx_peer[r] + k.part_off : part_peer[r];
        xa.dx.p[r] = dx_peer[r] + (size_t)k.r0 * H * 2;
        xa.flags.p[r] = cm->p2p_peer[r];
      }
      xa.rowstat = rs + k.r0;
      xa.mybuf = cm->p2p_buf;
      xa.g = g;
      xa.rank = cm->rank;
      xa.s0 = (int)(k.rows * cm->rank / g);
      xa.s1 = (int)(k.rows * (cm->rank + 1) / g);
      xa.H = (int)H;
      xa.epoch = dx_ep[i];
      cudaStream_t xs = cm->cs ? cm->cs : c.s;
      if (xs != c.s) {
        SLF_CUDA(cudaEventRecord(cm->ev_in, c.s));
        SLF_CUDA(cudaStreamWaitEvent(xs, cm->ev_in, 0));
      }
      const int blocks = 8 * std::max(8, tl_reserved_sms);  // 8 resident blocks per reserved SM
      p2p_dx_exchange_kernel<<<blocks, 256, 0, xs>>>(xa);
      SLF_CUDA(cudaGetLastError());
    } else if (dX) {
      SLF_TRY(comm_allreduce_start(cm, dxp, (size_t)k.rows * H, 0, c.s));
      pending = (int64_t)i;
    }
  }
  if (p2p_dx && !chunks.empty()) {  // every rank's slices of every chunk are in this rank's dhidden
    SLF_TRY(p2p_wait(cm, (int)P2P_DX_DONE_OFF, dx_ep[chunks.size() - 1], c.s));
    if (cm->cs) {
      SLF_CUDA(cudaEventRecord(cm->ev_ag, cm->cs));
      SLF_CUDA(cudaStreamWaitEvent(c.s, cm->ev_ag, 0));
    }
  }
  if (pending >= 0) SLF_TRY(finish());
  SLF_TRY(s_end(c, a, reduction, scale, loss_out, dW));
  if (cm->p2p && cm->p2p_buf) {  // a timed-out wait poisons this call's loss and fails the next call
    const int64_t n_loss = reduction == SLF_NONE ? N : 1;
    p2p_check_kernel<<<(int)std::min<int64_t>((n_loss + 255) / 256, 64), 256, 0, c.s>>>(cm->p2p_buf, loss_out, n_loss,
                                                                                      cm->p2p_err_dev);
    SLF_CUDA(cudaGetLastError());
  }
  return SLF_OK;
}

// ---- final RMSNorm fused into schedule S (slf_rmsnorm_lce_fwd_bwd) ------------------
// Workspace: [ schedule-S workspace (planner budget b) | 2 y chunk buffers [max chunk rows][H] bf16 |
// rstd [N] fp32 | 2 dg partial buffers [max chunk rows / RMS_RG][H] fp32 ].  With budget 0 the LCE part takes its
// default 5 % plan and the RMSNorm buffers come on top; otherwise the whole layout fits `budget`.
struct RmsPlan {
  Plan p;
  size_t off_y0, off_y1, off_rstd, off_part0, off_part1, total;
};

bool rms_layout(int64_t N, int64_t H, int64_t V, size_t b, RmsPlan* rp) {
  if (!plan_s(N, H, V, b, &rp->p)) return false;
  int64_t ymax = 0;
  for (const SChunk& k : s_chunks(rp->p, N, H, true, nullptr)) ymax = std::max(ymax, k.rows);
  const size_t yb = (size_t)ymax * H * 2, pb = (size_t)((ymax + RMS_RG - 1) / RMS_RG) * H * 4;
  rp->off_y0 = align_up(rp->p.total, 1024);
  rp->off_y1 = align_up(rp->off_y0 + yb, 1024);
  rp->off_rstd = align_up(rp->off_y1 + yb, 1024);
  rp->off_part0 = align_up(rp->off_rstd + (size_t)N * 4, 1024);
  rp->off_part1 = align_up(rp->off_part0 + pb, 1024);
  rp->total = rp->off_part1 + pb;
  return true;
}

bool rms_plan(int64_t N, int64_t H, int64_t V, size_t budget, RmsPlan* out) {
  if (N < 1 || H < 8 || V < 1) return false;
  if (budget == 0) return rms_layout(N, H, V, 0, out);
  // The largest LCE budget whose whole layout fits (bisection): below the smallest feasible LCE plan
  // the predicate counts as "go larger", above it the layout grows with the budget.
  RmsPlan rp;
  auto below_or_fits = [&](size_t b) { return !rms_layout(N, H, V, b, &rp) || rp.total <= budget; };
  size_t lo = 1, hi = budget;
  while (lo < hi) {
    const size_t mid = lo + (hi - lo + 1) / 2;
    if (below_or_fits(mid))
      lo = mid;
    else
      hi = mid - 1;
  }
  if (!rms_layout(N, H, V, lo, &rp) || rp.total > budget) return false;
  *out = rp;
  return true;
}

}  // namespace

// ---- C ABI ---------------------------------------------------------------------------------------
extern "C" {

int slf_lce_version(void) { return 100; }

const char* slf_last_error_string(void) { return g_err.c_str(); }

size_t slf_lce_workspace_bytes(int64_t N, int64_t H, int64_t V_local, int schedule, size_t budget_bytes) {
  Plan r, s;
  const bool has_r = plan_r(N, H, V_local, budget_bytes, &r);
  const bool has_s = plan_s(N, H, V_local, budget_bytes, &s);
  switch (schedule) {
    case SLF_SCHED_R: return has_r ? r.total : 0;
    case SLF_SCHED_S: return has_s ? s.total : 0;
    case SLF_SCHED_AUTO: return std::max(has_r ? r.total : 0, has_s ? s.total : 0);
    default: return 0;
  }
}

slf_status slf_lce_plan_describe(int64_t N, int64_t H, int64_t V_local, int schedule, size_t budget_bytes, char* out,
                                 size_t cap) {
  if (!out || cap == 0) return fail(SLF_ERR_ARG, "null output buffer");
  if (schedule < SLF_SCHED_AUTO || schedule > SLF_SCHED_S) return fail(SLF_ERR_ARG, "schedule %d", schedule);
  Plan p;
  if (!plan_any(N, H, V_local, schedule, budget_bytes, true, &p)) return fail(SLF_ERR_WORKSPACE, "no plan fits");
  if (p.sched == SLF_SCHED_S) {
    const std::vector<SChunk> ch = s_chunks(p, N, H, true, nullptr);
    const int64_t fused = (int64_t)ch.size();
    int64_t rescaled = 0;  // chunks without room for X'^T: the in-place rescale, a combine launch of their own
    for (const SChunk& k : ch) {
      const size_t lo = align_up((size_t)(k.r0 + k.rows) * H * 2 + (size_t)k.ext * p.ld_stash * 2, 1024);
      rescaled += lo + (size_t)H * ((k.rows + 7) / 8 * 8) * 2 > (size_t)N * H * 2;
    }
    snprintf(out, cap,
             "schedule=S row_chunk=%lld n_chunks=%lld fused_chunks_with_dhidden=%lld rescaled_chunks=%lld "
             "stash_bytes=%zu workspace=%zu launches=%lld",
             (long long)p.C, (long long)p.nCh, (long long)fused, (long long)rescaled, (size_t)p.C * p.ld_stash * 2,
             p.total, (long long)(8 + fused * 2 + rescaled));
  } else {
    snprintf(out, cap,
             "schedule=R row_block=%lld n_row_blocks=%lld vocab_chunk=%lld n_vocab_chunks=%lld workspace=%zu "
             "fwd_partials=%zu bwd=%zu launches=%lld",
             (long long)p.R, (long long)p.nR, (long long)p.Cv, (long long)p.nC, p.total, p.fwd_bytes, p.bwd_bytes,
             (long long)(4 + p.nR * p.nC * 2));
  }
  return SLF_OK;
}

slf_status slf_lce_fwd_bwd(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                           int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                           void* dhidden, void* dweight, void* workspace, size_t workspace_bytes, int schedule,
                           size_t budget_bytes, void* stream) {
  return slf_lce_fwd_bwd_ex(hidden, weight, targets, N, H, V, ignore_index, reduction, scale, loss_out, dhidden,
                            dweight, workspace, workspace_bytes, schedule, budget_bytes, 0u, stream);
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  if (!a || !b) return false;
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

// Outputs must not alias the inputs or the workspace (dhidden's unwritten rows are stash scratch).
slf_status check_outputs(const void* hidden, const void* weight, int64_t N, int64_t H, int64_t V, const void* dhidden,
                         const void* dweight, const void* workspace, size_t workspace_bytes) {
  const size_t xb = (size_t)N * H * 2, wb = (size_t)V * H * 2;
  if (overlaps(dhidden, xb, hidden, xb) || overlaps(dhidden, xb, weight, wb) ||
      overlaps(dhidden, xb, workspace, workspace_bytes) || overlaps(dhidden, xb, dweight, wb))
    return fail(SLF_ERR_ARG, "dhidden overlaps hidden, weight, dweight or the workspace");
  if (overlaps(dweight, wb, hidden, xb) || overlaps(dweight, wb, weight, wb) ||
      overlaps(dweight, wb, workspace, workspace_bytes))
    return fail(SLF_ERR_ARG, "dweight overlaps hidden, weight or the workspace");
  return SLF_OK;
}

slf_status slf_lce_fwd_bwd_ex(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                              int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                              void* dhidden, void* dweight, void* workspace, size_t workspace_bytes, int schedule,
                              size_t budget_bytes, uint32_t flags, void* stream) {
  SLF_TRY(check_common(hidden, weight, targets, N, H, V, workspace));
  SLF_TRY(check_outputs(hidden, weight, N, H, V, dhidden, dweight, workspace, workspace_bytes));
  if (flags & ~(uint32_t)SLF_FLAG_ACCUMULATE_DW) return fail(SLF_ERR_ARG, "unknown flags 0x%x", flags);
  if (!loss_out) return fail(SLF_ERR_ARG, "null loss_out");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if (schedule < SLF_SCHED_AUTO || schedule > SLF_SCHED_S) return fail(SLF_ERR_ARG, "schedule %d", schedule);
  if ((dhidden && !aligned16(dhidden)) || (dweight && !aligned16(dweight)))
    return fail(SLF_ERR_ALIGN, "gradient pointers must be 16-byte aligned");
  if (!aligned16(loss_out)) return fail(SLF_ERR_ALIGN, "loss_out must be 16-byte aligned");
  Ctx c;
  SLF_TRY(setup(c, N, H, V, budget_bytes, workspace, workspace_bytes, stream, schedule, true));
  c.acc_dw = (flags & SLF_FLAG_ACCUMULATE_DW) != 0;
  if (c.plan.sched == SLF_SCHED_S)
    return phase_s(c, hidden, weight, targets, N, H, V, ignore_index, reduction, scale, loss_out, dhidden, dweight);
  slf_shardstat* st = reinterpret_cast<slf_shardstat*>(c.ws + c.plan.off_shard);
  slf_rowstat* rs = reinterpret_cast<slf_rowstat*>(c.ws + c.plan.off_rowstat);
  SLF_TRY(phase_stats(c, hidden, weight, targets, N, H, V, 0, ignore_index, st));
  SLF_TRY(phase_combine(c, st, 1, targets, N, 0, V, V, ignore_index, reduction, scale, loss_out, rs));
  SLF_TRY(phase_backward(c, hidden, weight, rs, N, H, V, 1.0f, dhidden, 0, dweight));
  return SLF_OK;
}

std::mutex g_host_mu;  // serialises slf_lce_fwd_bwd_host enqueues (shared copy stream / events)

slf_status slf_lce_fwd_bwd_host(const void* hidden_host, const void* weight, const int32_t* targets_host, int64_t N,
                                int64_t H, int64_t V, int32_t ignore_index, int reduction, float scale,
                                float* loss_host, void* dhidden, void* dweight, void* hidden_dev,
                                int32_t* targets_dev, float* loss_dev, void* workspace, size_t workspace_bytes,
                                int schedule, size_t budget_bytes, uint32_t flags, void* stream) {
  if (!hidden_host || !targets_host || !loss_host) return fail(SLF_ERR_ARG, "null host pointer");
  SLF_TRY(check_common(hidden_dev, weight, targets_dev, N, H, V, workspace));
  SLF_TRY(check_outputs(hidden_dev, weight, N, H, V, dhidden, dweight, workspace, workspace_bytes));
  if (flags & ~(uint32_t)SLF_FLAG_ACCUMULATE_DW) return fail(SLF_ERR_ARG, "unknown flags 0x%x", flags);
  if (!loss_dev || !aligned16(loss_dev)) return fail(SLF_ERR_ALIGN, "loss_dev must be a 16-byte aligned pointer");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if (schedule < SLF_SCHED_AUTO || schedule > SLF_SCHED_S) return fail(SLF_ERR_ARG, "schedule %d", schedule);
  if ((dhidden && !aligned16(dhidden)) || (dweight && !aligned16(dweight)))
    return fail(SLF_ERR_ALIGN, "gradient pointers must be 16-byte aligned");
  std::lock_guard<std::mutex> hk(g_host_mu);
  Ctx c;
  SLF_TRY(setup(c, N, H, V, budget_bytes, workspace, workspace_bytes, stream, schedule, true));
  c.acc_dw = (flags & SLF_FLAG_ACCUMULATE_DW) != 0;
  DevInfo& d = *c.dev;
  if (!d.copy_stream) SLF_CUDA(cudaStreamCreateWithFlags(&d.copy_stream, cudaStreamNonBlocking));
  const size_t row_bytes = (size_t)H * 2;
  const uint8_t* hh = reinterpret_cast<const uint8_t*>(hidden_host);
  uint8_t* hd = reinterpret_cast<uint8_t*>(hidden_dev);
  SLF_CUDA(cudaMemcpyAsync(targets_dev, targets_host, (size_t)N * 4, cudaMemcpyHostToDevice, c.s));
  std::vector<SChunk> chunks;
  if (c.plan.sched == SLF_SCHED_S) chunks = s_chunks(c.plan, N, H, dhidden != nullptr, reinterpret_cast<uint8_t*>(dhidden));
  if (chunks.empty()) {  // schedule R: everything up front, in stream order
    SLF_CUDA(cudaMemcpyAsync(hd, hh, (size_t)N * row_bytes, cudaMemcpyHostToDevice, c.s));
  } else {
    while (d.copy_events.size() < chunks.size() + 1) {
      cudaEvent_t e;
      SLF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      d.copy_events.push_back(e);
    }
    // The staging buffer may still be read by an earlier call: wait for the end of the last call
    // that used it (tracked per staging pointer), else for everything already on `stream`.
    auto it = d.staging_free.find(hidden_dev);
    const cudaEvent_t free_ev = it != d.staging_free.end() ? it->second : d.copy_events[chunks.size()];
    if (it == d.staging_free.end()) SLF_CUDA(cudaEventRecord(free_ev, c.s));
    c.enqueue_inputs = [&d, free_ev, &chunks, hh, hd, row_bytes]() -> slf_status {
      SLF_CUDA(cudaStreamWaitEvent(d.copy_stream, free_ev, 0));
      for (size_t i = 0; i < chunks.size(); ++i) {
        const size_t off = (size_t)chunks[i].r0 * row_bytes;
        SLF_CUDA(cudaMemcpyAsync(hd + off, hh + off, (size_t)chunks[i].rows * row_bytes, cudaMemcpyHostToDevice,
                                 d.copy_stream));
        SLF_CUDA(cudaEventRecord(d.copy_events[i], d.copy_stream));
      }
      return SLF_OK;
    };
    c.chunk_ready = d.copy_events.data();
  }
  if (c.plan.sched == SLF_SCHED_S) {
    SLF_TRY(phase_s(c, hidden_dev, weight, targets_dev, N, H, V, ignore_index, reduction, scale, loss_dev, dhidden,
                    dweight));
  } else {
    slf_shardstat* st = reinterpret_cast<slf_shardstat*>(c.ws + c.plan.off_shard);
    slf_rowstat* rs = reinterpret_cast<slf_rowstat*>(c.ws + c.plan.off_rowstat);
    SLF_TRY(phase_stats(c, hidden_dev, weight, targets_dev, N, H, V, 0, ignore_index, st));
    SLF_TRY(phase_combine(c, st, 1, targets_dev, N, 0, V, V, ignore_index, reduction, scale, loss_dev, rs));
    SLF_TRY(phase_backward(c, hidden_dev, weight, rs, N, H, V, 1.0f, dhidden, 0, dweight));
  }
  SLF_CUDA(cudaMemcpyAsync(loss_host, loss_dev, (reduction == SLF_NONE ? (size_t)N : 1) * 4, cudaMemcpyDeviceToHost,
                           c.s));
  if (!chunks.empty()) {  // every reader of hidden_dev is enqueued: mark the staging buffer's release
    auto& ev = d.staging_free[hidden_dev];
    if (!ev) SLF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SLF_CUDA(cudaEventRecord(ev, c.s));
  }
  return SLF_OK;
}

slf_status slf_lce_fwd(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                       int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                       slf_rowstat* rowstat, void* workspace, size_t workspace_bytes, size_t budget_bytes,
                       void* stream) {
  SLF_TRY(check_common(hidden, weight, targets, N, H, V, workspace));
  if (!loss_out || !rowstat) return fail(SLF_ERR_ARG, "null loss_out/rowstat");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if (!aligned16(rowstat)) return fail(SLF_ERR_ALIGN, "rowstat must be 16-byte aligned");
  Ctx c;
  SLF_TRY(setup(c, N, H, V, budget_bytes, workspace, workspace_bytes, stream));
  slf_shardstat* st = reinterpret_cast<slf_shardstat*>(c.ws + c.plan.off_shard);
  SLF_TRY(phase_stats(c, hidden, weight, targets, N, H, V, 0, ignore_index, st));
  SLF_TRY(phase_combine(c, st, 1, targets, N, 0, V, V, ignore_index, reduction, scale, loss_out, rowstat));
  return SLF_OK;
}

slf_status slf_lce_fwd_shard_stats(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                                   int64_t H, int64_t V_local, int64_t vocab_start, int32_t ignore_index,
                                   slf_shardstat* shardstat, void* workspace, size_t workspace_bytes,
                                   size_t budget_bytes, void* stream) {
  SLF_TRY(check_common(hidden, weight_shard, targets, N, H, V_local, workspace));
  if (!shardstat) return fail(SLF_ERR_ARG, "null shardstat");
  if (!aligned16(shardstat)) return fail(SLF_ERR_ALIGN, "shardstat must be 16-byte aligned");
  if (vocab_start < 0) return fail(SLF_ERR_ARG, "vocab_start < 0");
  Ctx c;
  SLF_TRY(setup(c, N, H, V_local, budget_bytes, workspace, workspace_bytes, stream));
  SLF_TRY(phase_stats(c, hidden, weight_shard, targets, N, H, V_local, vocab_start, ignore_index, shardstat));
  return SLF_OK;
}

slf_status slf_lce_stats_combine(const slf_shardstat* stats, int g, const int32_t* targets, int64_t N,
                                 int64_t vocab_start, int64_t V_local, int64_t V_global, int32_t ignore_index,
                                 int reduction, float scale, float* loss_out, slf_rowstat* rowstat,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  if (!stats || !targets || !loss_out || !rowstat || !workspace) return fail(SLF_ERR_ARG, "null required pointer");
  if (g < 1 || N < 1 || V_local < 1 || V_global < 1 || vocab_start < 0 || vocab_start + V_local > V_global)
    return fail(SLF_ERR_ARG, "bad shard geometry");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if (!aligned16(stats) || !aligned16(targets) || !aligned16(rowstat) || !aligned16(workspace))
    return fail(SLF_ERR_ALIGN, "device pointers must be 16-byte aligned");
  if (workspace_bytes < WS_HEADER_BYTES) return fail(SLF_ERR_WORKSPACE, "workspace smaller than its header");
  Ctx c;
  SLF_TRY(device_info(&c.dev));
  c.s = reinterpret_cast<cudaStream_t>(stream);
  c.ws = reinterpret_cast<uint8_t*>(workspace);
  SLF_TRY(phase_combine(c, stats, g, targets, N, vocab_start, V_local, V_global, ignore_index, reduction, scale,
                        loss_out, rowstat));
  return SLF_OK;
}

slf_status slf_lce_bwd(const void* hidden, const void* weight, const int32_t* targets, const slf_rowstat* rowstat,
                       int64_t N, int64_t H, int64_t V_local, float grad_scale, void* dhidden, int dhidden_fp32,
                       void* dweight, void* workspace, size_t workspace_bytes, size_t budget_bytes, void* stream) {
  SLF_TRY(check_common(hidden, weight, targets, N, H, V_local, workspace));
  if (!rowstat) return fail(SLF_ERR_ARG, "null rowstat");
  if (!aligned16(rowstat) || (dhidden && !aligned16(dhidden)) || (dweight && !aligned16(dweight)))
    return fail(SLF_ERR_ALIGN, "device pointers must be 16-byte aligned");
  Ctx c;
  SLF_TRY(setup(c, N, H, V_local, budget_bytes, workspace, workspace_bytes, stream));
  SLF_TRY(phase_backward(c, hidden, weight, rowstat, N, H, V_local, grad_scale, dhidden, dhidden_fp32, dweight));
  return SLF_OK;
}

// ---- schedule S split (vocab shards) ----------------------------------------------------------------
static slf_status setup_s(Ctx& c, int64_t N, int64_t H, int64_t V_l, size_t budget, void* ws, size_t ws_bytes,
                          void* stream) {
  return setup(c, N, H, V_l, budget, ws, ws_bytes, stream, SLF_SCHED_S, true);
}

slf_status slf_lce_s_plan(int64_t N, int64_t H, int64_t V_local, size_t budget_bytes, int64_t* chunk_rows,
                          int64_t* n_chunks) {
  if (!chunk_rows || !n_chunks) return fail(SLF_ERR_ARG, "null output");
  Plan p;
  if (!plan_s(N, H, V_local, budget_bytes, &p)) return fail(SLF_ERR_WORKSPACE, "no schedule-S plan fits the budget");
  *chunk_rows = p.C;
  *n_chunks = p.nCh;
  return SLF_OK;
}

slf_status slf_lce_s_begin(const int32_t* targets, int64_t N, int64_t H, int64_t V_local, int64_t vocab_start,
                           int64_t V_global, int32_t ignore_index, int need_dweight, void* workspace,
                           size_t workspace_bytes, size_t budget_bytes, void* stream) {
  if (!targets || !workspace) return fail(SLF_ERR_ARG, "null required pointer");
  if (!aligned16(targets) || !aligned16(workspace)) return fail(SLF_ERR_ALIGN, "pointers must be 16-byte aligned");
  if (vocab_start < 0 || vocab_start + V_local > V_global) return fail(SLF_ERR_ARG, "bad shard geometry");
  Ctx c;
  SLF_TRY(setup_s(c, N, H, V_local, budget_bytes, workspace, workspace_bytes, stream));
  const SArgs a{nullptr, nullptr, targets, N, H, V_local, vocab_start, V_global, ignore_index};
  return s_begin(c, a, need_dweight != 0);
}

slf_status slf_lce_s_chunk_stats(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                                 int64_t H, int64_t V_local, int64_t vocab_start, int64_t V_global,
                                 int32_t ignore_index, int64_t chunk, slf_shardstat* shardstat_chunk, void* workspace,
                                 size_t workspace_bytes, size_t budget_bytes, void* stream) {
  SLF_TRY(check_common(hidden, weight_shard, targets, N, H, V_local, workspace));
  if (!shardstat_chunk || !aligned16(shardstat_chunk)) return fail(SLF_ERR_ARG, "bad shardstat_chunk");
  if (vocab_start < 0 || vocab_start + V_local > V_global) return fail(SLF_ERR_ARG, "bad shard geometry");
  Ctx c;
  SLF_TRY(setup_s(c, N, H, V_local, budget_bytes, workspace, workspace_bytes, stream));
  if (chunk < 0 || chunk >= c.plan.nCh) return fail(SLF_ERR_ARG, "chunk %lld out of range", (long long)chunk);
  const SArgs a{hidden, weight_shard, targets, N, H, V_local, vocab_start, V_global, ignore_index};
  return s_chunk_stats(c, a, s_plain_chunk(c.plan, N, chunk), shardstat_chunk);
}

slf_status slf_lce_s_chunk_bwd(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                               int64_t H, int64_t V_local, int64_t vocab_start, int64_t V_global,
                               int32_t ignore_index, int reduction, float scale, int64_t chunk,
                               const slf_shardstat* stats, int g, float* loss_rows, void* dhidden_chunk,
                               int dhidden_fp32, void* dweight, void* workspace, size_t workspace_bytes,
                               size_t budget_bytes, void* stream) {
  SLF_TRY(check_common(hidden, weight_shard, targets, N, H, V_local, workspace));
  if (!stats || g < 1 || !aligned16(stats)) return fail(SLF_ERR_ARG, "bad stats");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if (reduction == SLF_NONE && !loss_rows) return fail(SLF_ERR_ARG, "reduction NONE needs loss_rows");
  if ((dhidden_chunk && !aligned16(dhidden_chunk)) || (dweight && !aligned16(dweight)))
    return fail(SLF_ERR_ALIGN, "gradient pointers must be 16-byte aligned");
  Ctx c;
  SLF_TRY(setup_s(c, N, H, V_local, budget_bytes, workspace, workspace_bytes, stream));
  if (chunk < 0 || chunk >= c.plan.nCh) return fail(SLF_ERR_ARG, "chunk %lld out of range", (long long)chunk);
  const SArgs a{hidden, weight_shard, targets, N, H, V_local, vocab_start, V_global, ignore_index};
  float* lr = reduction == SLF_NONE ? loss_rows : reinterpret_cast<float*>(c.ws + c.plan.off_loss);
  return s_chunk_bwd(c, a, s_plain_chunk(c.plan, N, chunk), stats, g, reduction, scale, lr, dhidden_chunk,
                     dhidden_fp32, dweight);
}

slf_status slf_lce_s_end(const void* hidden, int64_t N, int64_t H, int64_t V_local, int reduction, float scale,
                         float* loss_out, void* dweight, void* workspace, size_t workspace_bytes, size_t budget_bytes,
                         void* stream) {
  if (!hidden || !workspace) return fail(SLF_ERR_ARG, "null required pointer");
  if (reduction != SLF_NONE && !loss_out) return fail(SLF_ERR_ARG, "null loss_out");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  Ctx c;
  SLF_TRY(setup_s(c, N, H, V_local, budget_bytes, workspace, workspace_bytes, stream));
  const SArgs a{hidden, nullptr, nullptr, N, H, V_local, 0, V_local, 0};
  return s_end(c, a, reduction, scale, loss_out, dweight);
}

slf_status slf_lce_s_rowstat(int64_t N, int64_t H, int64_t V_local, size_t budget_bytes, void* workspace,
                             const slf_rowstat** out) {
  if (!workspace || !out) return fail(SLF_ERR_ARG, "null pointer");
  Plan p;
  if (!plan_s(N, H, V_local, budget_bytes, &p)) return fail(SLF_ERR_WORKSPACE, "no schedule-S plan fits the budget");
  *out = reinterpret_cast<const slf_rowstat*>(reinterpret_cast<uint8_t*>(workspace) + p.off_rowstat);
  return SLF_OK;
}

// ---- communicator + vocab-sharded call ------------------------------------------------------------
slf_status slf_comm_get_unique_id(void* id128) {
  if (!id128) return fail(SLF_ERR_ARG, "null id buffer");
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(SLF_ERR_COMM, "%s", api.why);
  ncclUniqueId id;
  const ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return comm_fail_nccl(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id128, &id, 128);
  return SLF_OK;
}

static slf_status comm_events(slf_comm_s* c) {
  SLF_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  SLF_CUDA(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  SLF_CUDA(cudaEventCreateWithFlags(&c->ev_ag, cudaEventDisableTiming));
  for (auto& e : c->ev_ar) SLF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SLF_OK;
}

slf_status slf_comm_init(slf_comm* out, const void* id128, int rank, int world, int device) {
  if (!out || !id128) return fail(SLF_ERR_ARG, "null pointer");
  if (world < 1 || rank < 0 || rank >= world) return fail(SLF_ERR_ARG, "rank %d of world %d", rank, world);
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(SLF_ERR_COMM, "%s", api.why);
  SLF_CUDA(cudaSetDevice(device));
  slf_comm_s* c = new slf_comm_s;
  c->rank = rank;
  c->world = world;
  c->device = device;
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  slf_status st = comm_events(c);
  if (st == SLF_OK) {
    const ncclResult_t r = api.CommInitRank(&c->nccl, world, id, rank);
    if (r != ncclSuccess) st = comm_fail_nccl(r, "ncclCommInitRank");
  }
  if (st != SLF_OK) {
    slf_comm_destroy(c);
    return st;
  }
  *out = c;
  return SLF_OK;
}

slf_status slf_comm_init_callbacks(slf_comm* out, int rank, int world, slf_allgather_fn allgather,
                                   slf_allreduce_f32_fn allreduce, void* user) {
  if (!out || !allgather || !allreduce) return fail(SLF_ERR_ARG, "null pointer");
  if (world < 1 || rank < 0 || rank >= world) return fail(SLF_ERR_ARG, "rank %d of world %d", rank, world);
  slf_comm_s* c = new slf_comm_s;
  c->rank = rank;
  c->world = world;
  cudaGetDevice(&c->device);
  c->cb_allgather = allgather;
  c->cb_allreduce = allreduce;
  c->cb_user = user;
  *out = c;
  return SLF_OK;
}

slf_status slf_comm_destroy(slf_comm c) {
  if (!c) return SLF_OK;
  slf_status st = SLF_OK;
  p2p_release(c);
  if (c->nccl) {
    const ncclResult_t r = nccl_api().CommDestroy(c->nccl);
    if (r != ncclSuccess) st = comm_fail_nccl(r, "ncclCommDestroy");
  }
  if (c->cs) cudaStreamDestroy(c->cs);
  if (c->p2p_err_host) cudaFreeHost(c->p2p_err_host);
  for (cudaEvent_t e : {c->ev_in, c->ev_ag, c->ev_ar[0], c->ev_ar[1]})
    if (e) cudaEventDestroy(e);
  delete c;
  return st;
}

slf_status slf_comm_set_p2p(slf_comm c, int enable) {
  if (!c) return fail(SLF_ERR_ARG, "null communicator");
  if (enable < 0 || enable > 3) return fail(SLF_ERR_ARG, "P2P mode %d (bits: 1 statistics, 2 dX)", enable);
  if (enable && c->world > P2P_MAX_RANKS) return fail(SLF_ERR_ARG, "P2P supports <= %d ranks", P2P_MAX_RANKS);
  if (!enable) p2p_release(c);
  c->p2p = enable != 0;
  c->p2p_mode = enable;
  return SLF_OK;
}

slf_status slf_comm_status(slf_comm c, int32_t* p2p_timeouts) {
  if (!c || !p2p_timeouts) return fail(SLF_ERR_ARG, "null pointer");
  *p2p_timeouts = 0;
  if (c->p2p_buf) SLF_CUDA(cudaMemcpy(p2p_timeouts, c->p2p_buf + P2P_ERR_OFF, 4, cudaMemcpyDeviceToHost));
  if (c->p2p_err_host && *reinterpret_cast<volatile int*>(c->p2p_err_host)) *p2p_timeouts = 1;
  return SLF_OK;
}

slf_status slf_comm_rank(slf_comm c, int* rank, int* world) {
  if (!c || !rank || !world) return fail(SLF_ERR_ARG, "null pointer");
  *rank = c->rank;
  *world = c->world;
  return SLF_OK;
}

slf_status slf_shard_bounds(int64_t V_global, int world, int rank, int64_t* vocab_start, int64_t* V_local) {
  if (!vocab_start || !V_local) return fail(SLF_ERR_ARG, "null output");
  if (world < 1 || rank < 0 || rank >= world || V_global < world) return fail(SLF_ERR_ARG, "bad shard geometry");
  shard_bounds(V_global, world, rank, vocab_start, V_local);
  return SLF_OK;
}

size_t slf_lce_sharded_workspace_bytes(int64_t N, int64_t H, int64_t V_global, int world, int rank,
                                       size_t budget_bytes) {
  ShardPlan sp;
  return shard_plan(N, H, V_global, world, rank, budget_bytes, &sp) ? sp.total : 0;
}

slf_status slf_lce_sharded_plan_describe(int64_t N, int64_t H, int64_t V_global, int world, int rank,
                                         size_t budget_bytes, char* out, size_t cap) {
  if (!out || cap == 0) return fail(SLF_ERR_ARG, "null output buffer");
  ShardPlan sp;
  if (!shard_plan(N, H, V_global, world, rank, budget_bytes, &sp)) return fail(SLF_ERR_WORKSPACE, "no plan fits");
  const std::vector<SChunk> ch = shard_chunks(sp, N, H, V_global, world, true, nullptr);
  const size_t ext_chunks = ch.size();
  size_t n_top = 0, n_tail = 0;
  for (const SChunk& k : ch) {
    n_top += k.part_off >= 0;
    n_tail += k.part_off == PART_WS_TAIL;
  }
  snprintf(out, cap,
           "schedule=S sharded world=%d rank=%d vocab_start=%lld V_local=%lld row_chunk=%lld n_chunks=%lld "
           "chunks_with_dhidden=%zu dx_partial=%s tail_rows=%lld xt_tail=%d top_chunks=%zu tail_chunks=%zu planner_budget=%zu "
           "stash_bytes=%zu workspace=%zu",
           world, rank, (long long)sp.v0, (long long)sp.V_l, (long long)sp.p.C, (long long)sp.p.nCh, ext_chunks,
           sp.ws_part ? "workspace" : "dhidden_top", (long long)sp.r_tail, sp.xt_tail ? 1 : 0, n_top, n_tail, sp.b, (size_t)sp.p.C * sp.p.ld_stash * 2,
           sp.total);
  return SLF_OK;
}

slf_status slf_lce_sharded_chunk_table(int64_t N, int64_t H, int64_t V_global, int world, int rank,
                                       size_t budget_bytes, int64_t* out, int64_t cap, int64_t* n_chunks) {
  if (!n_chunks || (cap > 0 && !out)) return fail(SLF_ERR_ARG, "null output");
  ShardPlan sp;
  if (!shard_plan(N, H, V_global, world, rank, budget_bytes, &sp)) return fail(SLF_ERR_WORKSPACE, "no plan fits");
  const std::vector<SChunk> ch = shard_chunks(sp, N, H, V_global, world, true, nullptr);
  *n_chunks = (int64_t)ch.size();
  for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)ch.size()); ++i) {
    const SChunk& k = ch[i];
    const int64_t row[6] = {k.r0, k.rows, k.ext, k.part_off, (int64_t)k.xt_lim, shard_ld_max(V_global, world)};
    memcpy(out + 6 * i, row, sizeof(row));
  }
  return SLF_OK;
}

slf_status slf_lce_fwd_bwd_sharded(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                                   int64_t H, int64_t V_global, int32_t ignore_index, int reduction, float scale,
                                   float* loss_out, void* dhidden, void* dweight_shard, void* workspace,
                                   size_t workspace_bytes, size_t budget_bytes, slf_comm comm, void* stream) {
  if (!comm) return fail(SLF_ERR_ARG, "null communicator");
  if (comm->p2p_err_host && *reinterpret_cast<volatile int*>(comm->p2p_err_host))
    return fail(SLF_ERR_COMM, "a P2P wait of an earlier call on this communicator timed out (its loss is NaN); "
                              "recreate the communicator");
  if (V_global < comm->world) return fail(SLF_ERR_ARG, "V_global %lld < world %d", (long long)V_global, comm->world);
  int64_t v0, vl;
  shard_bounds(V_global, comm->world, comm->rank, &v0, &vl);
  SLF_TRY(check_common(hidden, weight_shard, targets, N, H, vl, workspace));
  SLF_TRY(check_outputs(hidden, weight_shard, N, H, vl, dhidden, dweight_shard, workspace, workspace_bytes));
  if (!loss_out || !aligned16(loss_out)) return fail(SLF_ERR_ALIGN, "loss_out must be a 16-byte aligned pointer");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if ((dhidden && !aligned16(dhidden)) || (dweight_shard && !aligned16(dweight_shard)))
    return fail(SLF_ERR_ALIGN, "gradient pointers must be 16-byte aligned");
  ShardPlan sp;
  if (!shard_plan(N, H, V_global, comm->world, comm->rank, budget_bytes, &sp))
    return fail(SLF_ERR_WORKSPACE, "no sharded schedule-S plan fits the budget");
  if (workspace_bytes < sp.total)
    return fail(SLF_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, sp.total);
  Ctx c;
  SLF_TRY(setup(c, N, H, vl, sp.b, workspace, sp.p.total, stream, SLF_SCHED_S, true));
  // SMs left to the communicator's kernels at world > 1 (SLF_COMM_SMS, default 8): leaving 4 / 8 of
  // the 148 SMs costs 0.4 / 1.3 % of a Llama-8B step under the power cap (world 1, forced), and it
  // lets NCCL's all-reduce blocks run beside the persistent GEMMs (not measurable on one GPU).
  static const int comm_sms = getenv("SLF_COMM_SMS") ? atoi(getenv("SLF_COMM_SMS")) : 8;
  ReserveSms reserve(comm->world > 1 || getenv("SLF_COMM_SMS_FORCE") ? comm_sms : 0);
  return phase_sharded(c, sp, comm, hidden, weight_shard, targets, N, H, V_global, ignore_index, reduction, scale,
                       loss_out, dhidden, dweight_shard);
}

slf_status slf_lce_fwd_bwd_dp(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                              int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                              void* dhidden, void* dweight, void* workspace, size_t workspace_bytes, int schedule,
                              size_t budget_bytes, int sync_dweight, slf_comm comm, void* stream) {
  if (!comm) return fail(SLF_ERR_ARG, "null communicator");
  if (sync_dweight && !comm->nccl && comm->world > 1)
    return fail(SLF_ERR_UNSUPPORTED, "sync_dweight needs the NCCL transport (bf16 all-reduce)");
  SLF_TRY(check_common(hidden, weight, targets, N, H, V, workspace));
  SLF_TRY(check_outputs(hidden, weight, N, H, V, dhidden, dweight, workspace, workspace_bytes));
  if (!loss_out || !aligned16(loss_out)) return fail(SLF_ERR_ALIGN, "loss_out must be a 16-byte aligned pointer");
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if (schedule < SLF_SCHED_AUTO || schedule > SLF_SCHED_S) return fail(SLF_ERR_ARG, "schedule %d", schedule);
  if ((dhidden && !aligned16(dhidden)) || (dweight && !aligned16(dweight)))
    return fail(SLF_ERR_ALIGN, "gradient pointers must be 16-byte aligned");
  Ctx c;
  SLF_TRY(setup(c, N, H, V, budget_bytes, workspace, workspace_bytes, stream, schedule, true));
  // scratch for the limbs: the header's spare words (WsHeader::pad)
  WsHeader* hdr = reinterpret_cast<WsHeader*>(hdr_of(c.ws));
  float* limbs = reinterpret_cast<float*>(&hdr->pad[0]);
  if (reduction == SLF_MEAN && comm->world > 1) {
    c.after_prep = [&]() -> slf_status {
      if (comm->nccl) {
        NcclApi& api = nccl_api();
        SLF_CUDA(cudaEventRecord(comm->ev_in, c.s));
        SLF_CUDA(cudaStreamWaitEvent(comm->cs, comm->ev_in, 0));
        ncclResult_t r;
        {
          ProfScope ps(SLF_PROF_COMM_ALLREDUCE, comm->cs, 0.0, 8.0);
          r = api.AllReduce(&hdr->n_valid, &hdr->n_valid, 1, ncclUint64, ncclSum, comm->nccl, comm->cs);
        }
        if (r != ncclSuccess) return comm_fail_nccl(r, "ncclAllReduce(n_valid)");
        SLF_CUDA(cudaEventRecord(comm->ev_ag, comm->cs));
        SLF_CUDA(cudaStreamWaitEvent(c.s, comm->ev_ag, 0));
        return SLF_OK;
      }
      u64_to_limbs_kernel<<<1, 1, 0, c.s>>>(&hdr->n_valid, limbs);
      SLF_CUDA(cudaGetLastError());
      SLF_TRY(comm_allreduce_now(comm, limbs, 3, c.s));
      limbs_to_u64_kernel<<<1, 1, 0, c.s>>>(limbs, &hdr->n_valid);
      SLF_CUDA(cudaGetLastError());
      return SLF_OK;
    };
  }
  if (c.plan.sched == SLF_SCHED_S) {
    SLF_TRY(phase_s(c, hidden, weight, targets, N, H, V, ignore_index, reduction, scale, loss_out, dhidden, dweight));
  } else {
    slf_shardstat* st = reinterpret_cast<slf_shardstat*>(c.ws + c.plan.off_shard);
    slf_rowstat* rs = reinterpret_cast<slf_rowstat*>(c.ws + c.plan.off_rowstat);
    SLF_TRY(phase_stats(c, hidden, weight, targets, N, H, V, 0, ignore_index, st));
    SLF_TRY(phase_combine(c, st, 1, targets, N, 0, V, V, ignore_index, reduction, scale, loss_out, rs));
    SLF_TRY(phase_backward(c, hidden, weight, rs, N, H, V, 1.0f, dhidden, 0, dweight));
  }
  if (comm->world > 1 && reduction != SLF_NONE) SLF_TRY(comm_allreduce_now(comm, loss_out, 1, c.s));
  if (sync_dweight && dweight && comm->world > 1) {  // the ordinary data-parallel gradient sync (bf16)
    NcclApi& api = nccl_api();
    SLF_CUDA(cudaEventRecord(comm->ev_in, c.s));
    SLF_CUDA(cudaStreamWaitEvent(comm->cs, comm->ev_in, 0));
    ncclResult_t r;
    {
      ProfScope ps(SLF_PROF_COMM_ALLREDUCE, comm->cs, 0.0, (double)V * H * 2);
      r = api.AllReduce(dweight, dweight, (size_t)V * H, ncclBfloat16, ncclSum, comm->nccl, comm->cs);
    }
    if (r != ncclSuccess) return comm_fail_nccl(r, "ncclAllReduce(dW)");
    SLF_CUDA(cudaEventRecord(comm->ev_ag, comm->cs));
    SLF_CUDA(cudaStreamWaitEvent(c.s, comm->ev_ag, 0));
  }
  return SLF_OK;
}

// Debug: how many clusters of `cluster` CTAs of the GEMM kernel (its smem footprint) fit at once.
slf_status slf_debug_max_active_clusters(int cluster, int* out) {
  if (!out || cluster < 1 || cluster > 16) return fail(SLF_ERR_ARG, "bad arguments");
  DevInfo* dev;
  SLF_TRY(device_info(&dev));
  auto kfn = lce_group_kernel<2, 4>;
  SLF_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<2, 4>::SMEM_BYTES));
  if (cluster > 8) SLF_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(dev->sms / cluster * cluster));
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Cfg<2, 4>::SMEM_BYTES;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SLF_CUDA(cudaOccupancyMaxActiveClusters(out, kfn, &cfg));
  return SLF_OK;
}

// ---- bf16 in-place scaling (autograd: apply grad_output to gradients formed in the forward) ----------
slf_status slf_scale_bf16(void* p, int64_t n, float s, void* stream) {
  if (!p || n < 0 || (n % 8)) return fail(SLF_ERR_ARG, "p must be non-null and n a multiple of 8");
  if (!aligned16(p)) return fail(SLF_ERR_ALIGN, "pointer must be 16-byte aligned");
  DevInfo* dev;
  SLF_TRY(device_info(&dev));
  if (n == 0) return SLF_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t groups = n / 8;
  const int blocks = (int)std::min<int64_t>((groups + 255) / 256, (int64_t)dev->sms * 8);
  scale_bf16_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<uint4*>(p), groups, s);
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

slf_status slf_scale_bf16_dev(void* p, int64_t n, const float* s_dev, void* stream) {
  if (!p || !s_dev || n < 0 || (n % 8)) return fail(SLF_ERR_ARG, "p, s must be non-null and n a multiple of 8");
  if (!aligned16(p)) return fail(SLF_ERR_ALIGN, "pointer must be 16-byte aligned");
  DevInfo* dev;
  SLF_TRY(device_info(&dev));
  if (n == 0) return SLF_OK;
  const int64_t groups = n / 8;
  const int blocks = (int)std::min<int64_t>((groups + 255) / 256, (int64_t)dev->sms * 8);
  scale_bf16_dev_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(reinterpret_cast<uint4*>(p), groups,
                                                                                   s_dev);
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

slf_status slf_rowstat_scale(const slf_rowstat* in, const float* grad, int per_row, int64_t N, slf_rowstat* out,
                             void* stream) {
  if (!in || !grad || !out || N < 1) return fail(SLF_ERR_ARG, "null pointer or N < 1");
  if (!aligned16(in) || !aligned16(out)) return fail(SLF_ERR_ALIGN, "rowstat pointers must be 16-byte aligned");
  rowstat_scale_kernel<<<(unsigned)((N + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(in), grad, per_row, N, reinterpret_cast<float4*>(out));
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

// ---- debug trace (SLF_DEBUG_TRACE) ------------------------------------------------------------------
slf_status slf_debug_trace_read(uint64_t* host, int64_t n) {
  if (!host || n < 0) return fail(SLF_ERR_ARG, "bad arguments");
  n = std::min<int64_t>(n, (int64_t)(TRACE_TILES + TRACE_UNITS) * 8);
  SLF_CUDA(cudaDeviceSynchronize());
  SLF_CUDA(cudaMemcpyFromSymbol(host, g_trace, (size_t)n * 8));
  return SLF_OK;
}

// ---- final RMSNorm (NEXT-1) ---------------------------------------------------------------------------
static int rms_rows_per_block(DevInfo* dev, int64_t N) {
  const int64_t blocks = std::max<int64_t>(1, 2 * (int64_t)dev->sms);
  return (int)std::max<int64_t>(1, (N + blocks - 1) / blocks);
}

size_t slf_rmsnorm_workspace_bytes(int64_t N, int64_t H) {
  if (N < 1 || H < 8) return 0;
  const int64_t blocks = 2 * 148 + 64;  // upper bound on the grid for any B200 SM count
  (void)N;
  return (size_t)blocks * H * 4;
}

slf_status slf_rmsnorm_fwd(const void* x, const void* g, int64_t N, int64_t H, float eps, void* y, float* rstd,
                           void* stream) {
  if (!x || !g || !y || !rstd) return fail(SLF_ERR_ARG, "null pointer");
  if (N < 1 || H < 8 || H % 8 || H > 16384) return fail(SLF_ERR_ARG, "bad sizes (H %% 8 == 0, H <= 16384)");
  if (!aligned16(x) || !aligned16(g) || !aligned16(y) || !aligned16(rstd))
    return fail(SLF_ERR_ALIGN, "pointers must be 16-byte aligned");
  DevInfo* dev;
  SLF_TRY(device_info(&dev));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ProfScope ps(SLF_PROF_RMSNORM, s, 0.0, (double)N * H * 4 + N * 4.0);
  rmsnorm_fwd_kernel<<<(unsigned)N, RMS_THREADS, 0, s>>>(reinterpret_cast<const uint16_t*>(x),
                                                         reinterpret_cast<const uint16_t*>(g), H, eps,
                                                         reinterpret_cast<uint16_t*>(y), rstd);
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

slf_status slf_rmsnorm_bwd(const void* x, const void* g, const float* rstd, const void* dy, int64_t N, int64_t H,
                           void* dx, float* dg, void* workspace, size_t workspace_bytes, void* stream) {
  if (!x || !g || !rstd || !dy || !dx || !dg || !workspace) return fail(SLF_ERR_ARG, "null pointer");
  if (N < 1 || H < 8 || H % 8 || H > 16384) return fail(SLF_ERR_ARG, "bad sizes (H %% 8 == 0, H <= 16384)");
  if (!aligned16(x) || !aligned16(g) || !aligned16(rstd) || !aligned16(dy) || !aligned16(dx) || !aligned16(workspace))
    return fail(SLF_ERR_ALIGN, "pointers must be 16-byte aligned");
  DevInfo* dev;
  SLF_TRY(device_info(&dev));
  const int rpb = rms_rows_per_block(dev, N);
  const int blocks = (int)((N + rpb - 1) / rpb);
  if (workspace_bytes < (size_t)blocks * H * 4) return fail(SLF_ERR_WORKSPACE, "rmsnorm workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float* part = reinterpret_cast<float*>(workspace);
  {
    ProfScope ps(SLF_PROF_RMSNORM, s, 0.0, (double)N * H * 8 + (double)blocks * H * 4);
    const size_t smem = (size_t)H * 4;
    if (smem > 48 * 1024)
      SLF_CUDA(cudaFuncSetAttribute(rmsnorm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rmsnorm_bwd_kernel<<<(unsigned)blocks, RMS_THREADS, smem, s>>>(
        reinterpret_cast<const uint16_t*>(x), reinterpret_cast<const uint16_t*>(g), rstd,
        reinterpret_cast<const uint16_t*>(dy), N, H, rpb, reinterpret_cast<uint16_t*>(dx), part);
    SLF_CUDA(cudaGetLastError());
    rmsnorm_dg_reduce_kernel<<<(unsigned)((H + 255) / 256), 256, 0, s>>>(part, blocks, H, dg);
    SLF_CUDA(cudaGetLastError());
  }
  return SLF_OK;
}

size_t slf_rmsnorm_lce_workspace_bytes(int64_t N, int64_t H, int64_t V, size_t budget_bytes) {
  RmsPlan rp;
  return rms_plan(N, H, V, budget_bytes, &rp) ? rp.total : 0;
}

slf_status slf_rmsnorm_lce_fwd_bwd(const void* x, const void* g, float eps, const void* weight, const int32_t* targets,
                                   int64_t N, int64_t H, int64_t V, int32_t ignore_index, int reduction, float scale,
                                   float* loss_out, void* dx, float* dg, void* dweight, void* workspace,
                                   size_t workspace_bytes, size_t budget_bytes, void* stream) {
  SLF_TRY(check_common(x, weight, targets, N, H, V, workspace));
  if (!g || !dx || !dg || !dweight || !loss_out) return fail(SLF_ERR_ARG, "null pointer (g, dx, dg, dweight, loss)");
  if (!aligned16(g) || !aligned16(dx) || !aligned16(dg) || !aligned16(dweight) || !aligned16(loss_out))
    return fail(SLF_ERR_ALIGN, "pointers must be 16-byte aligned");
  if (H > 16384) return fail(SLF_ERR_ARG, "H %lld > 16384", (long long)H);
  if (reduction < SLF_SUM || reduction > SLF_NONE) return fail(SLF_ERR_ARG, "bad reduction %d", reduction);
  if (!(eps >= 0.f)) return fail(SLF_ERR_ARG, "eps must be >= 0");
  SLF_TRY(check_outputs(x, weight, N, H, V, dx, dweight, workspace, workspace_bytes));
  RmsPlan rp;
  if (!rms_plan(N, H, V, budget_bytes, &rp)) return fail(SLF_ERR_WORKSPACE, "no schedule-S plan fits the budget");
  if (workspace_bytes < rp.total)
    return fail(SLF_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, rp.total);
  Ctx c;
  SLF_TRY(device_info(&c.dev));
  c.plan = rp.p;
  c.s = reinterpret_cast<cudaStream_t>(stream);
  c.ws = reinterpret_cast<uint8_t*>(workspace);
  RmsFuse rf{};
  rf.g = g;
  rf.eps = eps;
  rf.dg = dg;
  rf.ybuf[0] = c.ws + rp.off_y0;
  rf.ybuf[1] = c.ws + rp.off_y1;
  rf.rstd = reinterpret_cast<float*>(c.ws + rp.off_rstd);
  rf.part[0] = reinterpret_cast<float*>(c.ws + rp.off_part0);
  rf.part[1] = reinterpret_cast<float*>(c.ws + rp.off_part1);
  rf.mref = reinterpret_cast<float*>(c.ws + rp.p.off_mref);
  return phase_s(c, x, weight, targets, N, H, V, ignore_index, reduction, scale, loss_out, dx, dweight, &rf);
}

slf_status slf_rmsnorm_lce_plan_describe(int64_t N, int64_t H, int64_t V, size_t budget_bytes, char* out, size_t cap) {
  if (!out || cap == 0) return fail(SLF_ERR_ARG, "null output buffer");
  RmsPlan rp;
  if (!rms_plan(N, H, V, budget_bytes, &rp)) return fail(SLF_ERR_WORKSPACE, "no plan fits");
  snprintf(out, cap, "schedule=S rmsnorm_fused row_chunk=%lld n_chunks=%lld lce_workspace=%zu y_chunk_bytes=%zu "
                     "workspace=%zu", (long long)rp.p.C, (long long)rp.p.nCh, rp.p.total, rp.off_y1 - rp.off_y0, rp.total);
  return SLF_OK;
}

slf_status slf_lce_status(const void* workspace, void* stream, int32_t* bad_targets, int64_t* n_valid) {
  if (!workspace || !bad_targets) return fail(SLF_ERR_ARG, "null pointer");
  SLF_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  WsHeader h;
  SLF_CUDA(cudaMemcpy(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost));
  *bad_targets = h.bad;
  if (n_valid) *n_valid = (int64_t)h.n_valid;
  return SLF_OK;
}

// scratch: counts [V_l + 2] | hit rows [min(N, V_l)] | span totals | packed sort keys
static void csr_scratch_layout(int64_t N, int64_t V_l, size_t* o_hits, size_t* o_bsum, size_t* o_sort, size_t* total) {
  *o_hits = align_up((size_t)(V_l + 2) * 4, 256);
  *o_bsum = align_up(*o_hits + (size_t)std::min(N, V_l) * 4, 256);
  *o_sort = align_up(*o_bsum + (size_t)((V_l + CSR_SCAN_SPAN - 1) / CSR_SCAN_SPAN) * 8, 256);
  *total = *o_sort + csr_sort_bytes(N);
}

size_t slf_target_csr_scratch_bytes(int64_t N, int64_t V_local) {
  if (N < 1 || V_local < 1) return 0;
  size_t a, b, c, t;
  csr_scratch_layout(N, V_local, &a, &b, &c, &t);
  return t;
}

slf_status slf_target_csr(const int32_t* targets, int64_t N, int32_t ignore_index, int64_t vocab_start,
                          int64_t V_local, int32_t* offsets, int32_t* token_idx, void* scratch, size_t scratch_bytes,
                          void* stream) {
  if (!targets || !offsets || !token_idx || !scratch) return fail(SLF_ERR_ARG, "null pointer");
  if (N < 1 || V_local < 1 || vocab_start < 0 || N > (1ll << 31) - 1 || V_local >= (1ll << 20))
    return fail(SLF_ERR_ARG, "bad sizes N=%lld V_local=%lld", (long long)N, (long long)V_local);
  if (!aligned16(targets) || !aligned16(scratch)) return fail(SLF_ERR_ALIGN, "targets / scratch must be 16-byte aligned");
  size_t o_hits, o_bsum, o_sort, total;
  csr_scratch_layout(N, V_local, &o_hits, &o_bsum, &o_sort, &total);
  if (scratch_bytes < total) return fail(SLF_ERR_WORKSPACE, "scratch %zu bytes < required %zu", scratch_bytes, total);
  uint8_t* sc = reinterpret_cast<uint8_t*>(scratch);
  int32_t* cnt = reinterpret_cast<int32_t*>(sc);
  return build_csr(reinterpret_cast<cudaStream_t>(stream), targets, N, ignore_index, vocab_start, V_local, cnt, offsets,
                   reinterpret_cast<int32_t*>(sc + o_hits), token_idx, reinterpret_cast<int2*>(sc + o_bsum),
                   o_sort - o_bsum, sc + o_sort, total - o_sort);
}

slf_status slf_lce_dx_finalize(const float* dhidden_fp32, const slf_rowstat* rowstat, void* dhidden, int64_t N,
                               int64_t H, void* stream) {
  if (!dhidden_fp32 || !rowstat || !dhidden) return fail(SLF_ERR_ARG, "null pointer");
  if (N < 1 || H < 8 || H % 8) return fail(SLF_ERR_ARG, "bad sizes");
  if (!aligned16(dhidden_fp32) || !aligned16(rowstat) || !aligned16(dhidden))
    return fail(SLF_ERR_ALIGN, "pointers must be 16-byte aligned");
  DevInfo* dev;
  SLF_TRY(device_info(&dev));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t groups = N * H / 8;
  const int blocks = (int)std::min<int64_t>((groups + 255) / 256, (int64_t)dev->sms * 8);
  ProfScope ps(SLF_PROF_DX_FINALIZE, s, 0.0, (double)N * H * 6 + N * 16.0);
  dx_finalize_kernel<<<blocks, 256, 0, s>>>(dhidden_fp32, rowstat, reinterpret_cast<uint16_t*>(dhidden), N, H);
  SLF_CUDA(cudaGetLastError());
  return SLF_OK;
}

slf_status slf_profile_begin(void) {
  for (auto& r : g_prof.recs) {
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.recs.clear();
  g_prof.on = true;
  return SLF_OK;
}

slf_status slf_profile_end(double* ms, int64_t* launches, double* flops, double* bytes) {
  g_prof.on = false;
  for (int k = 0; k < SLF_PROF_KINDS; ++k) {
    if (ms) ms[k] = 0;
    if (launches) launches[k] = 0;
    if (flops) flops[k] = 0;
    if (bytes) bytes[k] = 0;
  }
  for (auto& r : g_prof.recs) {
    SLF_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    SLF_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    if (ms) ms[r.kind] += t;
    if (launches) launches[r.kind] += 1;
    if (flops) flops[r.kind] += r.flops;
    if (bytes) bytes[r.kind] += r.bytes;
  }
  return SLF_OK;
}

slf_status slf_debug_gemm(const void* A, const void* B, float* D, int64_t M, int64_t N, int64_t K, int a_mn,
                          int b_mn, void* stream) {
  if (!A || !B || !D) return fail(SLF_ERR_ARG, "null pointer");
  if (M < 8 || N < 8 || K < 8 || M % 8 || N % 8 || K % 8) return fail(SLF_ERR_ARG, "M, N, K must be multiples of 8");
  if (!aligned16(A) || !aligned16(B) || !aligned16(D)) return fail(SLF_ERR_ALIGN, "pointers must be 16-byte aligned");
  DevInfo* dev;
  SLF_TRY(device_info(&dev));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CUtensorMap ta, tb;
  if (a_mn)
    SLF_TRY(tmap_mnmajor(&ta, A, M, K, M));
  else
    SLF_TRY(tmap_kmajor(&ta, A, K, M, K, BM));
  if (b_mn)
    SLF_TRY(tmap_mnmajor(&tb, B, N, K, N, b_box_rows() / 64));
  else
    SLF_TRY(tmap_kmajor(&tb, B, K, N, K, b_box_rows()));
  GemmArgs a{};
  a.M = (int)M;
  a.N = (int)N;
  a.K = (int)K;
  a.out = D;
  a.ld_out = N;
  if (!a_mn && !b_mn) return launch_gemm<EPI_F32, false, false>(dev, ta, tb, a, s);
  if (!a_mn && b_mn) return launch_gemm<EPI_F32, false, true>(dev, ta, tb, a, s);
  if (a_mn && !b_mn) return launch_gemm<EPI_F32, true, false>(dev, ta, tb, a, s);
  return launch_gemm<EPI_F32, true, true>(dev, ta, tb, a, s);
}

}  // extern "C"
