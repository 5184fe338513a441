"""One fine-tuning step of the LM-head block, end to end (PAPER.md l.137, l.219,
l.231-237, l.273): the final RMSNorm and the fused linear-cross-entropy forward + backward in ONE
library call (slf_rmsnorm_lce_fwd_bwd: loss, dx, dg, dW; no [N x V] logits, no [N x H] normalised
activations), then Layer-Adam on the host for the head's weight, fed from the device
(slf_adam_step_device_async: dW chunks d2h, AVX-512 update on the host as each lands, bf16 W chunks
h2d — PAPER.md l.137 "Asynchronous Parameter Updating", l.219 "Layer-Adam").

The step never reads a device value on the host: the loss stays on the device (read it when you
need it), and the next step's forward waits on the previous update through a stream wait
(slf_adam_wait), not a host synchronisation of the compute stream.

This module is orchestration only: every FLOP of the step runs in libslf_lce.so (CUDA kernels for
the LCE / RMSNorm, C++ for the host Adam update).
"""
from __future__ import annotations

import torch

from .adam import LayerAdam
from .lce import REDUCTIONS, rmsnorm_lce_fwd_bwd, rmsnorm_lce_workspace_bytes


class LMHeadTrainer:
    """Trains the LM head W [V, H] (bf16 on the device, fp32 master + Adam moments on the host) under a
    fixed final-RMSNorm weight g [H]; every step also returns dx (the gradient for the layers below)
    and dg.

        tr = LMHeadTrainer(W, g, lr=1e-4)
        for x, t in batches:
            loss, dx, dg = tr.step(x, t)   # x [N, H] bf16, t [N] int32 on the device
        tr.finish()                        # the last update has landed in W
    """

    def __init__(self, W: torch.Tensor, g: torch.Tensor, lr: float = 1e-4, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, adamw: bool = True, rms_eps: float = 1e-5, ignore_index: int = -100,
                 reduction: str = "mean", budget_bytes: int = 0, threads: int = 0):
        if not (W.is_cuda and g.is_cuda) or W.dtype != torch.bfloat16 or g.dtype != torch.bfloat16:
            raise TypeError("W and g must be bf16 CUDA tensors")
        if reduction not in REDUCTIONS or reduction == "none":
            raise ValueError("reduction must be 'mean' or 'sum' for a training step")
        self.W, self.g = W, g.contiguous()
        self.V, self.H = W.shape
        self.rms_eps, self.ignore_index, self.reduction, self.budget = rms_eps, ignore_index, reduction, budget_bytes
        self.adam = LayerAdam(W.numel(), lr=lr, betas=betas, eps=eps, weight_decay=weight_decay, adamw=adamw,
                              threads=threads)
        self.adam.set_params(W.detach().cpu())  # master weights = the bf16 values exactly
        self._bufs = {}
        self._pending = False
        self.steps = 0

    def _buffers(self, N: int):
        b = self._bufs.get(N)
        if b is None:
            dev = self.W.device
            b = dict(loss=torch.empty(1, dtype=torch.float32, device=dev),
                     dx=torch.empty(N, self.H, dtype=torch.bfloat16, device=dev),
                     dg=torch.empty(self.H, dtype=torch.float32, device=dev),
                     dW=torch.empty_like(self.W),
                     ws=torch.empty(rmsnorm_lce_workspace_bytes(N, self.H, self.V, self.budget), dtype=torch.uint8,
                                    device=dev))
            self._bufs = {N: b}  # one batch shape at a time (the workspace is sized for it)
        return b

    def step(self, x: torch.Tensor, targets: torch.Tensor, events=None):
        """One step on the batch (x, targets): returns (loss [1] fp32, dx, dg) as device tensors —
        the trainer's own buffers, rewritten by the next step() (clone them to keep them).  The
        dW of this step is being applied to W when it returns; the next step (or finish()) waits.
        `events` (optional pair of CUDA events) are recorded around the fused call (timing)."""
        b = self._buffers(x.shape[0])
        if self._pending:  # the forward reads W: the previous update's h2d copies first (stream wait)
            self.adam.wait(self.W.device)
            self._pending = False
        if events is not None:
            events[0].record()
        # dx / dW buffers are rewritten by this call: the previous update must have read its dW
        loss, dx, dg, dW = rmsnorm_lce_fwd_bwd(x, self.g, self.W, targets, eps=self.rms_eps,
                                               ignore_index=self.ignore_index, reduction=self.reduction,
                                               budget_bytes=self.budget, workspace=b["ws"],
                                               out=(b["loss"], b["dx"], b["dg"], b["dW"]))
        if events is not None:
            events[1].record()
        self.adam.step_device_async(dW, self.W)
        self._pending = True
        self.steps += 1
        return b["loss"], dx, dg

    def finish(self):
        if self._pending:
            self.adam.wait(self.W.device)
            self._pending = False

    def master(self):
        """(p, m, v, t) of the host optimizer (fp32 CPU tensors, step count)."""
        self.finish()
        return self.adam.state()

    def close(self):
        self.finish()
        self.adam.close()
