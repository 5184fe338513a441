// layer_adam.cpp — Layer-Adam on the host for the LM head's weight.
//
// PAPER.md l.219 (§3.2 "Layer-Adam Optimizer"): "A self-developed variant of DeepSpeed's CPU-Adam, it
// stores the optimizer states of each layer in a flattened tensor in the host memory.  When the
// gradients of the layer are offloaded to the CPU, the optimizer updates the layer's parameters
// separately."  PAPER.md l.137 (§3.1 "Asynchronous Parameter Updating"): gradients go d2h
// asynchronously and the CPU updates P_i while the GPU keeps computing.
//
// Here: one flat fp32 master copy p and moments m, v per parameter tensor (64-byte aligned host
// memory), an AVX-512 update (16 lanes; runtime-dispatched, a scalar loop of the same operation
// order otherwise) split over OpenMP threads, and a device-fed step that pipelines, chunk by chunk,
// the bf16 gradient's device->host copy, the CPU update of the chunks that have landed and the
// host->device copy of the updated bf16 parameters (three overlapping stages).
// Update (reading R11; DeepSpeed CPU-Adam / torch.optim.AdamW), per element, fp32:
//   g = grad_scale * bf16(grad);  p *= 1 - lr*wd (adamw)  |  g += wd*p (L2)
//   m = b1*m + (1-b1)*g;  v = b2*v + (1-b2)*g*g
//   p -= (lr / (1 - b1^t)) * m / (sqrt(v) / sqrt(1 - b2^t) + eps);   out = RNE_bf16(p)
// No fused multiply-adds (built with -ffp-contract=off, intrinsics use separate mul/add), so the
// AVX-512 and scalar paths give identical bits.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/slf_adam.h"

namespace {

thread_local std::string g_adam_err;

slf_status afail(slf_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_adam_err = buf;
  return s;
}

#define ADAM_CUDA(x)                                                                          \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) return afail(SLF_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

struct Coef {
  float gs, decay, wd, b1, omb1, b2, omb2, inv_sqrt_bc2, eps, step;
  bool adamw;
};

inline uint16_t bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;  // NaN
  return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

void update_scalar(const Coef& c, float* p, float* m, float* v, const uint16_t* g16, uint16_t* out, int64_t i0,
                   int64_t i1) {
  for (int64_t i = i0; i < i1; ++i) {
    const uint32_t gb = (uint32_t)g16[i] << 16;
    float g;
    memcpy(&g, &gb, 4);
    g = g * c.gs;
    float pi = p[i];
    if (c.adamw)
      pi = pi * c.decay;
    else
      g = g + c.wd * pi;
    const float mi = c.b1 * m[i] + c.omb1 * g;
    const float vi = c.b2 * v[i] + c.omb2 * (g * g);
    const float den = std::sqrt(vi) * c.inv_sqrt_bc2 + c.eps;
    pi = pi - c.step * (mi / den);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (out) out[i] = bf16_rne(pi);
  }
}

__attribute__((target("avx512f,avx512bw"))) void update_avx512(const Coef& c, float* p, float* m, float* v,
                                                                const uint16_t* g16, uint16_t* out, int64_t i0,
                                                                int64_t i1) {
  const __m512 gs = _mm512_set1_ps(c.gs), decay = _mm512_set1_ps(c.decay), wd = _mm512_set1_ps(c.wd);
  const __m512 b1 = _mm512_set1_ps(c.b1), omb1 = _mm512_set1_ps(c.omb1), b2 = _mm512_set1_ps(c.b2),
               omb2 = _mm512_set1_ps(c.omb2), isb = _mm512_set1_ps(c.inv_sqrt_bc2), eps = _mm512_set1_ps(c.eps),
               step = _mm512_set1_ps(c.step);
  const __m512i rbias = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1), absmask = _mm512_set1_epi32(0x7fffffff),
                inf = _mm512_set1_epi32(0x7f800000), qnan = _mm512_set1_epi32(0x7fc0);
  int64_t i = i0;
  for (; i + 16 <= i1; i += 16) {
    const __m256i gb = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(g16 + i));
    __m512 g = _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(gb), 16));
    g = _mm512_mul_ps(g, gs);
    __m512 pi = _mm512_loadu_ps(p + i);
    if (c.adamw)
      pi = _mm512_mul_ps(pi, decay);
    else
      g = _mm512_add_ps(g, _mm512_mul_ps(wd, pi));
    const __m512 mi = _mm512_add_ps(_mm512_mul_ps(b1, _mm512_loadu_ps(m + i)), _mm512_mul_ps(omb1, g));
    const __m512 vi = _mm512_add_ps(_mm512_mul_ps(b2, _mm512_loadu_ps(v + i)), _mm512_mul_ps(omb2, _mm512_mul_ps(g, g)));
    const __m512 den = _mm512_add_ps(_mm512_mul_ps(_mm512_sqrt_ps(vi), isb), eps);
    pi = _mm512_sub_ps(pi, _mm512_mul_ps(step, _mm512_div_ps(mi, den)));
    _mm512_storeu_ps(p + i, pi);
    _mm512_storeu_ps(m + i, mi);
    _mm512_storeu_ps(v + i, vi);
    if (out) {
      const __m512i u = _mm512_castps_si512(pi);
      __m512i r = _mm512_srli_epi32(_mm512_add_epi32(_mm512_add_epi32(u, rbias), _mm512_and_si512(_mm512_srli_epi32(u, 16), one)), 16);
      const __mmask16 nan = _mm512_cmpgt_epu32_mask(_mm512_and_si512(u, absmask), inf);
      r = _mm512_mask_mov_epi32(r, nan, qnan);
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + i), _mm512_cvtepi32_epi16(r));
    }
  }
  update_scalar(c, p, m, v, g16, out, i, i1);
}

bool has_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                         getenv("SLF_ADAM_NO_AVX512") == nullptr;
  return ok;
}

float* alloc_f32(int64_t n) {
  void* p = nullptr;
  if (posix_memalign(&p, 64, (size_t)std::max<int64_t>(n, 1) * 4) != 0) return nullptr;
  memset(p, 0, (size_t)std::max<int64_t>(n, 1) * 4);
  return static_cast<float*>(p);
}

}  // namespace

struct slf_adam_s {
  int64_t n = 0, t = 0;
  float *p = nullptr, *m = nullptr, *v = nullptr;
  slf_adam_config cfg{};
  int device = 0;
  // device-fed pipeline (created on first use)
  uint16_t *g_stage = nullptr, *p_stage = nullptr;  // pinned host bf16
  cudaStream_t d2h = nullptr, h2d = nullptr;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  int64_t chunk = 0;
  std::thread worker;
  bool busy = false, had_device_step = false, pipeline_ready = false;
  slf_status worker_status = SLF_OK;
  std::string worker_err;
};

namespace {

Coef coef_for(const slf_adam_s& a, int64_t t, float grad_scale) {
  const slf_adam_config& c = a.cfg;
  Coef k;
  k.gs = grad_scale;
  k.decay = 1.0f - c.lr * c.weight_decay;
  k.wd = c.weight_decay;
  k.b1 = c.beta1;
  k.omb1 = 1.0f - c.beta1;
  k.b2 = c.beta2;
  k.omb2 = 1.0f - c.beta2;
  const double bc1 = 1.0 - std::pow((double)c.beta1, (double)t), bc2 = 1.0 - std::pow((double)c.beta2, (double)t);
  k.inv_sqrt_bc2 = (float)(1.0 / std::sqrt(bc2));
  k.eps = c.eps;
  k.step = (float)(c.lr / bc1);
  k.adamw = c.adamw != 0;
  return k;
}

int threads_of(const slf_adam_s& a) { return a.cfg.threads > 0 ? a.cfg.threads : omp_get_max_threads(); }

// Elements [i0, i1) over the OpenMP team, 64-byte aligned blocks of 4096 elements.
void update_range(const slf_adam_s& a, const Coef& c, const uint16_t* g, uint16_t* out, int64_t i0, int64_t i1) {
  constexpr int64_t BLK = 4096;
  const int64_t nb = (i1 - i0 + BLK - 1) / BLK;
  const bool vec = has_avx512();
#pragma omp parallel for schedule(static) num_threads(threads_of(a))
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t s = i0 + b * BLK, e = std::min(i1, s + BLK);
    if (vec)
      update_avx512(c, a.p, a.m, a.v, g, out, s, e);
    else
      update_scalar(c, a.p, a.m, a.v, g, out, s, e);
  }
}

slf_status check_cfg(const slf_adam_config* c) {
  if (!c) return afail(SLF_ERR_ARG, "null config");
  if (!(c->lr >= 0) || !(c->beta1 >= 0 && c->beta1 < 1) || !(c->beta2 >= 0 && c->beta2 < 1) || !(c->eps > 0) ||
      !(c->weight_decay >= 0))
    return afail(SLF_ERR_ARG, "bad hyper-parameters (lr %g b1 %g b2 %g eps %g wd %g)", c->lr, c->beta1, c->beta2,
                 c->eps, c->weight_decay);
  return SLF_OK;
}

void release_pipeline(slf_adam_s* a) {
  if (a->g_stage) cudaFreeHost(a->g_stage);
  if (a->p_stage) cudaFreeHost(a->p_stage);
  if (a->d2h) cudaStreamDestroy(a->d2h);
  if (a->h2d) cudaStreamDestroy(a->h2d);
  if (a->ev_start) cudaEventDestroy(a->ev_start);
  if (a->ev_done) cudaEventDestroy(a->ev_done);
  for (auto e : a->ev_chunk)
    if (e) cudaEventDestroy(e);
  a->g_stage = a->p_stage = nullptr;
  a->d2h = a->h2d = nullptr;
  a->ev_start = a->ev_done = nullptr;
  a->ev_chunk.clear();
  a->pipeline_ready = false;
}

// Creates the device-fed pipeline on first use.  `pipeline_ready` is set only once every resource
// exists; a failure part-way releases what was created, so the next call retries from scratch
// instead of running on a half-built pipeline.
slf_status ensure_pipeline(slf_adam_s* a) {
  if (a->pipeline_ready) return SLF_OK;
  release_pipeline(a);
  auto fail_release = [a](cudaError_t e, const char* what) {
    const slf_status st = afail(SLF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    release_pipeline(a);
    return st;
  };
#define PIPE_TRY(call)                                   \
  do {                                                   \
    const cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return fail_release(e_, #call); \
  } while (0)
  PIPE_TRY(cudaGetDevice(&a->device));
  PIPE_TRY(cudaHostAlloc(reinterpret_cast<void**>(&a->g_stage), (size_t)a->n * 2, cudaHostAllocDefault));
  PIPE_TRY(cudaHostAlloc(reinterpret_cast<void**>(&a->p_stage), (size_t)a->n * 2, cudaHostAllocDefault));
  PIPE_TRY(cudaStreamCreateWithFlags(&a->d2h, cudaStreamNonBlocking));
  PIPE_TRY(cudaStreamCreateWithFlags(&a->h2d, cudaStreamNonBlocking));
  PIPE_TRY(cudaEventCreateWithFlags(&a->ev_start, cudaEventDisableTiming));
  PIPE_TRY(cudaEventCreateWithFlags(&a->ev_done, cudaEventDisableTiming));
  a->chunk = a->cfg.chunk_elems > 0 ? a->cfg.chunk_elems : (int64_t)16 << 20;
  const int64_t nch = (a->n + a->chunk - 1) / a->chunk;
  a->ev_chunk.assign((size_t)nch, nullptr);
  for (auto& e : a->ev_chunk) PIPE_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
#undef PIPE_TRY
  a->pipeline_ready = true;
  return SLF_OK;
}

}  // namespace

extern "C" {

const char* slf_adam_last_error_string(void) { return g_adam_err.c_str(); }

int slf_adam_simd_width(void) { return has_avx512() ? 16 : 1; }

slf_status slf_adam_create(slf_adam* out, int64_t n, const slf_adam_config* cfg) {
  if (!out || n < 1) return afail(SLF_ERR_ARG, "null output or n < 1");
  const slf_status s = check_cfg(cfg);
  if (s != SLF_OK) return s;
  slf_adam_s* a = new slf_adam_s;
  a->n = n;
  a->cfg = *cfg;
  a->p = alloc_f32(n);
  a->m = alloc_f32(n);
  a->v = alloc_f32(n);
  if (!a->p || !a->m || !a->v) {
    slf_adam_destroy(a);
    return afail(SLF_ERR_ARG, "cannot allocate 3 x %lld fp32 host states", (long long)n);
  }
  *out = a;
  return SLF_OK;
}

slf_status slf_adam_destroy(slf_adam a) {
  if (!a) return SLF_OK;
  if (a->worker.joinable()) a->worker.join();
  free(a->p);
  free(a->m);
  free(a->v);
  release_pipeline(a);
  delete a;
  return SLF_OK;
}

slf_status slf_adam_set_config(slf_adam a, const slf_adam_config* cfg) {
  if (!a) return afail(SLF_ERR_ARG, "null handle");
  if (a->busy) return afail(SLF_ERR_ARG, "a device-fed step is in flight (call slf_adam_wait)");
  const slf_status s = check_cfg(cfg);
  if (s != SLF_OK) return s;
  const int64_t keep_chunk = a->cfg.chunk_elems;
  a->cfg = *cfg;
  if (a->pipeline_ready) a->cfg.chunk_elems = keep_chunk;  // the pipeline's chunking is fixed once created
  return SLF_OK;
}

slf_status slf_adam_set_params(slf_adam a, const float* p_f32, const uint16_t* p_bf16) {
  if (!a || (!p_f32 && !p_bf16)) return afail(SLF_ERR_ARG, "null argument");
  if (a->busy) return afail(SLF_ERR_ARG, "a device-fed step is in flight");
  if (p_f32) {
    memcpy(a->p, p_f32, (size_t)a->n * 4);
  } else {
    for (int64_t i = 0; i < a->n; ++i) {
      const uint32_t u = (uint32_t)p_bf16[i] << 16;
      memcpy(&a->p[i], &u, 4);
    }
  }
  memset(a->m, 0, (size_t)a->n * 4);
  memset(a->v, 0, (size_t)a->n * 4);
  a->t = 0;
  return SLF_OK;
}

slf_status slf_adam_get_state(slf_adam a, float* p, float* m, float* v, int64_t* t) {
  if (!a) return afail(SLF_ERR_ARG, "null handle");
  if (a->busy) return afail(SLF_ERR_ARG, "a device-fed step is in flight");
  if (p) memcpy(p, a->p, (size_t)a->n * 4);
  if (m) memcpy(m, a->m, (size_t)a->n * 4);
  if (v) memcpy(v, a->v, (size_t)a->n * 4);
  if (t) *t = a->t;
  return SLF_OK;
}

slf_status slf_adam_step_host(slf_adam a, const uint16_t* grad_bf16, float grad_scale, uint16_t* param_bf16_out) {
  if (!a || !grad_bf16) return afail(SLF_ERR_ARG, "null argument");
  if (a->busy) return afail(SLF_ERR_ARG, "a device-fed step is in flight");
  a->t += 1;
  const Coef c = coef_for(*a, a->t, grad_scale);
  update_range(*a, c, grad_bf16, param_bf16_out, 0, a->n);
  return SLF_OK;
}

slf_status slf_adam_step_device_async(slf_adam a, const void* grad_bf16_dev, float grad_scale, void* param_bf16_dev,
                                      void* stream) {
  if (!a || !grad_bf16_dev || !param_bf16_dev) return afail(SLF_ERR_ARG, "null argument");
  if (a->busy) return afail(SLF_ERR_ARG, "a device-fed step is already in flight (call slf_adam_wait)");
  slf_status s = ensure_pipeline(a);
  if (s != SLF_OK) return s;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  // Both copy streams start after the work already on the caller's stream (the gradient's producer,
  // and the last reader of the parameters).
  ADAM_CUDA(cudaEventRecord(a->ev_start, cs));
  ADAM_CUDA(cudaStreamWaitEvent(a->d2h, a->ev_start, 0));
  ADAM_CUDA(cudaStreamWaitEvent(a->h2d, a->ev_start, 0));
  const uint8_t* gd = static_cast<const uint8_t*>(grad_bf16_dev);
  const int64_t nch = (int64_t)a->ev_chunk.size();
  for (int64_t k = 0; k < nch; ++k) {
    const int64_t i0 = k * a->chunk, i1 = std::min(a->n, i0 + a->chunk);
    ADAM_CUDA(cudaMemcpyAsync(a->g_stage + i0, gd + i0 * 2, (size_t)(i1 - i0) * 2, cudaMemcpyDeviceToHost, a->d2h));
    ADAM_CUDA(cudaEventRecord(a->ev_chunk[(size_t)k], a->d2h));
  }
  a->t += 1;
  const Coef c = coef_for(*a, a->t, grad_scale);
  a->busy = true;
  a->worker_status = SLF_OK;
  uint8_t* pd = static_cast<uint8_t*>(param_bf16_dev);
  const bool prev = a->had_device_step;
  a->had_device_step = true;
  a->worker = std::thread([a, c, pd, nch, prev]() {
    auto wfail = [a](const char* what, cudaError_t e) {
      a->worker_status = SLF_ERR_CUDA;
      a->worker_err = std::string(what) + ": " + cudaGetErrorString(e);
    };
    cudaError_t e = cudaSetDevice(a->device);
    if (e != cudaSuccess) return wfail("cudaSetDevice", e);
    // the previous step's last host->device copies read p_stage: let them finish before rewriting it
    if (prev && (e = cudaEventSynchronize(a->ev_done)) != cudaSuccess) return wfail("cudaEventSynchronize", e);
    for (int64_t k = 0; k < nch; ++k) {
      const int64_t i0 = k * a->chunk, i1 = std::min(a->n, i0 + a->chunk);
      if ((e = cudaEventSynchronize(a->ev_chunk[(size_t)k])) != cudaSuccess) return wfail("cudaEventSynchronize", e);
      update_range(*a, c, a->g_stage, a->p_stage, i0, i1);
      if ((e = cudaMemcpyAsync(pd + i0 * 2, a->p_stage + i0, (size_t)(i1 - i0) * 2, cudaMemcpyHostToDevice,
                               a->h2d)) != cudaSuccess)
        return wfail("cudaMemcpyAsync h2d", e);
    }
    if ((e = cudaEventRecord(a->ev_done, a->h2d)) != cudaSuccess) return wfail("cudaEventRecord", e);
  });
  return SLF_OK;
}

slf_status slf_adam_wait(slf_adam a, void* stream) {
  if (!a) return afail(SLF_ERR_ARG, "null handle");
  if (!a->busy) return SLF_OK;
  a->worker.join();
  a->busy = false;
  if (a->worker_status != SLF_OK) return afail(a->worker_status, "%s", a->worker_err.c_str());
  ADAM_CUDA(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), a->ev_done, 0));
  return SLF_OK;
}

}  // extern "C"
