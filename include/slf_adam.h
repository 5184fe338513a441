/*
 * slf_adam.h — C ABI of Layer-Adam, the host optimizer step for the LM head's weight
 * (SURVEY.md §8(f) NEXT-4), exported by the same libslf_lce.so.
 *
 * PAPER.md line 219 (§3.2 "Layer-Adam Optimizer"): "A self-developed variant of DeepSpeed's
 * CPU-Adam, it stores the optimizer states of each layer in a flattened tensor in the host memory.
 * When the gradients of the layer are offloaded to the CPU, the optimizer updates the layer's
 * parameters separately."  PAPER.md line 137 (§3.1 "Asynchronous Parameter Updating"): the
 * gradients are transferred d2h asynchronously while "the CPU applies the optimizer to update P_i
 * using the host-resident optimizer states" and the GPU keeps computing.
 *
 * The update (reading R11: DeepSpeed CPU-Adam = torch.optim.AdamW semantics), per
 * element, in fp32, step t = 1, 2, ...:
 *   g = grad_scale * grad;   p *= 1 - lr*wd  (adamw != 0)   |   g += wd * p  (adamw == 0, L2)
 *   m = b1*m + (1-b1)*g;     v = b2*v + (1-b2)*g*g
 *   p -= lr/(1-b1^t) * m / (sqrt(v)/sqrt(1-b2^t) + eps);     param_bf16 = RNE_bf16(p)
 * State: one flat fp32 master copy p and moments m, v of n elements in host memory, owned by the
 * handle.  Conventions: status codes and SLF_* values of slf_lce.h; the message of the last error
 * on this thread is slf_adam_last_error_string().  One call at a time per handle.
 */
#ifndef SLF_ADAM_H_
#define SLF_ADAM_H_

#include <stddef.h>
#include <stdint.h>

#include "slf_lce.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct slf_adam_s* slf_adam;

typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  int32_t adamw;       /* 1: decoupled weight decay (AdamW, DeepSpeed default); 0: L2 into g */
  int32_t threads;     /* OpenMP threads for the update (0: the OpenMP default) */
  int64_t chunk_elems; /* device-fed pipeline granularity (0: 16 Mi elements); fixed at first use */
} slf_adam_config;

const char* slf_adam_last_error_string(void);
/* 16 when the AVX-512 update runs on this host, 1 for the scalar loop (same operation order,
 * identical results). */
int slf_adam_simd_width(void);

/* A handle with n parameters, p = m = v = 0 and t = 0.  SLF_ERR_ARG on bad hyper-parameters
 * (lr < 0, beta outside [0, 1), eps <= 0, weight_decay < 0) or n < 1. */
slf_status slf_adam_create(slf_adam* out, int64_t n, const slf_adam_config* cfg);
slf_status slf_adam_destroy(slf_adam a);
/* New hyper-parameters (e.g. a learning-rate schedule) for the following steps. */
slf_status slf_adam_set_config(slf_adam a, const slf_adam_config* cfg);
/* Master parameters from HOST fp32 [n] (p_f32) or HOST bf16 bits [n] (p_bf16, widened exactly);
 * resets m, v and t. */
slf_status slf_adam_set_params(slf_adam a, const float* p_f32, const uint16_t* p_bf16);
/* HOST copies of p, m, v ([n] fp32 each; any may be NULL) and the step count t. */
slf_status slf_adam_get_state(slf_adam a, float* p, float* m, float* v, int64_t* t);

/* One step from a HOST bf16 gradient [n]; writes the HOST bf16 parameters [n] if param_bf16_out is
 * not NULL.  Synchronous. */
slf_status slf_adam_step_host(slf_adam a, const uint16_t* grad_bf16, float grad_scale, uint16_t* param_bf16_out);

/* One step fed from the DEVICE (the LCE's dW): after the work already enqueued on `stream`, the
 * bf16 gradient [n] (DEVICE, 16-byte aligned) is copied to pinned host staging chunk by chunk on
 * an internal stream; a host worker thread updates each chunk as it lands and copies its bf16
 * parameters back into param_bf16_dev [n] (DEVICE) on a second internal stream, so the three
 * stages overlap.  Returns once the copies are enqueued and the worker started.  Until
 * slf_adam_wait returns, neither device buffer may be reused (the gradient is being read, the
 * parameters written).  The first call allocates 2*n*2 bytes of pinned host staging. */
slf_status slf_adam_step_device_async(slf_adam a, const void* grad_bf16_dev, float grad_scale, void* param_bf16_dev,
                                      void* stream);
/* Joins the worker and makes `stream` wait for the last parameter copy (no-op when no step is in
 * flight).  Returns the worker's status. */
slf_status slf_adam_wait(slf_adam a, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SLF_ADAM_H_ */
