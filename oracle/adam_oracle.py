"""Plain CPU oracle for Layer-Adam on the LM head's weight.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
oracle legs may import this module; the product (``paper_2603_16428_b200``, its host C++
``csrc/layer_adam.cpp``) never imports it and shares no code with it.

What it computes.  PAPER.md l.219 (§3.2 "Layer-Adam Optimizer"): "A self-developed variant of
DeepSpeed's CPU-Adam, it stores the optimizer states of each layer in a flattened tensor in the host
memory.  When the gradients of the layer are offloaded to the CPU, the optimizer updates the
layer's parameters separately"; PAPER.md l.137 (§3.1 "Asynchronous Parameter Updating"): gradients
are transferred d2h asynchronously and "the CPU applies the optimizer to update P_i using the
host-resident optimizer states".  The paper writes no formula; DeepSpeed's CPU-Adam is Adam
(Kingma & Ba) with bias correction and, in its default adamw_mode, decoupled weight decay
(Loshchilov & Hutter), the same update as ``torch.optim.AdamW`` (reading R11).  Per step
t = 1, 2, ... on every element, in this order (float64 here):

    g      = grad_scale * grad                                  (grad: the bf16 dW, exact in fp64)
    p      = p * (1 - lr * wd)              if adamw (decoupled decay)
    g      = g + wd * p                     if not adamw (L2 mode, DeepSpeed adamw_mode=False)
    m      = b1 * m + (1 - b1) * g
    v      = b2 * v + (1 - b2) * g * g
    p      = p - (lr / (1 - b1^t)) * m / (sqrt(v) / sqrt(1 - b2^t) + eps)
    param_bf16 = RNE_bf16(p)                (the copy the GPU uses next step)

Pinned by tests/test_oracle_pins.py (torch.optim.AdamW / Adam float64 as an independent library
routine, the first-step closed form lr*g/(|g|+eps), the zero-gradient pure-decay closed form,
and the bias-corrected constant-gradient limit).
"""
from __future__ import annotations

import numpy as np


def adam_step(p, m, v, grad, t: int, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8,
              wd: float = 0.0, adamw: bool = True, grad_scale: float = 1.0):
    """One Layer-Adam step (t >= 1) on float64 copies; returns (p, m, v) new arrays."""
    if t < 1:
        raise ValueError("step t starts at 1")
    p = np.array(p, dtype=np.float64)
    m = np.array(m, dtype=np.float64)
    v = np.array(v, dtype=np.float64)
    g = grad_scale * np.asarray(grad, dtype=np.float64)
    if adamw:
        p = p * (1.0 - lr * wd)
    else:
        g = g + wd * p
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    bc1 = 1.0 - b1 ** t
    bc2 = 1.0 - b2 ** t
    p = p - (lr / bc1) * m / (np.sqrt(v) / np.sqrt(bc2) + eps)
    return p, m, v


def adam_steps(p0, grads, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8, wd: float = 0.0,
               adamw: bool = True, grad_scale: float = 1.0):
    """T steps from zero moments; grads is a sequence of T gradient arrays.  Returns (p, m, v,
    updates) with updates[t] = max |p_{t} - p_{t-1}| (used to derive the fp32 tolerance)."""
    p = np.array(p0, dtype=np.float64)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    ups = []
    for t, g in enumerate(grads, start=1):
        pn, m, v = adam_step(p, m, v, g, t, lr, b1, b2, eps, wd, adamw, grad_scale)
        ups.append(float(np.max(np.abs(pn - p))) if p.size else 0.0)
        p = pn
    return p, m, v, ups


def bf16_rne(x) -> np.ndarray:
    """Round float64 values to bf16 (round to nearest, ties to even) via float32: returns the
    uint16 bit patterns.  Float64 -> float32 is itself RNE; the float32 -> bf16 step is done on the
    bits.  (Double rounding is harmless for values exactly representable in float32, which is what
    the fp32-master comparison uses; the oracle's own p64 is compared within one bf16 ulp.)"""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16).astype(np.uint16)
    nan = np.isnan(f)
    if nan.any():
        r[nan] = 0x7FC0
    return r
