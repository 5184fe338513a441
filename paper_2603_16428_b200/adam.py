"""Layer-Adam: the host optimizer step for the LM head's weight, a thin
binding over include/slf_adam.h (C++/OpenMP/AVX-512 in libslf_lce.so).
("Layer-Adam Optimizer": DeepSpeed-CPU-Adam variant, flat host states per layer) and l.137
(gradients d2h asynchronously, CPU update overlapping GPU work)."""
from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib


class AdamConfig(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float), ("adamw", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("chunk_elems", ctypes.c_int64)]


def _acheck(status: int, what: str):
    if status != 0:
        from ._lib import STATUS_NAMES, SlfError
        msg = lib().slf_adam_last_error_string().decode(errors="replace")
        raise SlfError(f"{what} failed with {STATUS_NAMES.get(status, status)}: {msg}")


def simd_width() -> int:
    return int(lib().slf_adam_simd_width())


class LayerAdam:
    """Flat fp32 master weights + Adam moments in host memory for one parameter tensor of n elements.

    step_host(grad_bf16_cpu) — synchronous host step; step_device_async(grad_dev, param_dev) +
    wait() — the device-fed pipelined step (d2h of the gradient, CPU update, h2d of the bf16
    parameters, chunk by chunk)."""

    def __init__(self, n: int, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0,
                 adamw: bool = True, threads: int = 0, chunk_elems: int = 0):
        self.n = int(n)
        self.cfg = AdamConfig(lr, betas[0], betas[1], eps, weight_decay, int(adamw), threads, chunk_elems)
        h = ctypes.c_void_p(0)
        _acheck(lib().slf_adam_create(ctypes.byref(h), self.n, ctypes.byref(self.cfg)), "slf_adam_create")
        self.h = h.value

    def set_lr(self, lr: float):
        self.cfg.lr = lr
        _acheck(lib().slf_adam_set_config(self.h, ctypes.byref(self.cfg)), "slf_adam_set_config")

    def set_params(self, p):
        """Master weights from a CPU fp32 or bf16 tensor of n elements (resets moments and t)."""
        p = p.detach().reshape(-1).contiguous()
        if p.is_cuda:
            p = p.cpu()
        if p.numel() != self.n:
            raise ValueError(f"expected {self.n} elements, got {p.numel()}")
        if p.dtype == torch.float32:
            _acheck(lib().slf_adam_set_params(self.h, p.data_ptr(), None), "slf_adam_set_params")
        elif p.dtype == torch.bfloat16:
            _acheck(lib().slf_adam_set_params(self.h, None, p.data_ptr()), "slf_adam_set_params")
        else:
            raise TypeError("params must be float32 or bfloat16")

    def state(self):
        """(p, m, v) fp32 CPU tensors and t."""
        p, m, v = (torch.empty(self.n, dtype=torch.float32) for _ in range(3))
        t = ctypes.c_int64(0)
        _acheck(lib().slf_adam_get_state(self.h, p.data_ptr(), m.data_ptr(), v.data_ptr(), ctypes.byref(t)),
                "slf_adam_get_state")
        return p, m, v, t.value

    def step_host(self, grad_bf16, grad_scale: float = 1.0, out_bf16=None):
        if grad_bf16.dtype != torch.bfloat16 or grad_bf16.is_cuda or not grad_bf16.is_contiguous():
            raise TypeError("grad must be a contiguous CPU bf16 tensor")
        if grad_bf16.numel() != self.n:
            raise ValueError("gradient size mismatch")
        _acheck(lib().slf_adam_step_host(self.h, grad_bf16.data_ptr(), float(grad_scale),
                                         None if out_bf16 is None else out_bf16.data_ptr()), "slf_adam_step_host")
        return out_bf16

    def step_device_async(self, grad_dev, param_dev, grad_scale: float = 1.0):
        for t in (grad_dev, param_dev):
            if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous() or t.numel() != self.n:
                raise TypeError("grad and param must be contiguous CUDA bf16 tensors of n elements")
        s = torch.cuda.current_stream(grad_dev.device).cuda_stream
        _acheck(lib().slf_adam_step_device_async(self.h, grad_dev.data_ptr(), float(grad_scale), param_dev.data_ptr(),
                                                 s), "slf_adam_step_device_async")

    def wait(self, device=None):
        s = torch.cuda.current_stream(device).cuda_stream if torch.cuda.is_available() else None
        _acheck(lib().slf_adam_wait(self.h, s), "slf_adam_wait")

    def close(self):
        if getattr(self, "h", None):
            lib().slf_adam_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass
