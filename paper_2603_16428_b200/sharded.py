"""Vocab-sharded LCE across GPUs of one box (BASELINE.json north_star).

Rank k of a process group of size g owns LM-head rows [V*k//g, V*(k+1)//g).  One step:

    st_k   = shard_stats(X, W_k, t, v0_k)              per-row (m, s, z_t, hit) of the local vocab
    ST     = all_gather(st_k)  (rank order)            16 B/token per rank over NCCL / NVLink
    loss, rs_k = stats_combine(ST, t, v0_k, V_k, V)    deterministic shard-order merge
    dX_k, dW_k = lce_bwd(X, W_k, t, rs_k, fp32 dX)     recompute per tile; dW stays local
    dX     = all_reduce(sum_k dX_k)                    fp32 N*H*4 over NCCL
    dX_bf16 = dx_finalize(dX, rs_k)

Every compute step is a libslf_lce.so kernel; this module only orders the calls and the two
collectives.  The ops are injectable so the orchestration can be tested with world_size 2 on CPU
(gloo) against the oracle (tests/test_sharded_cpu.py).
"""
from __future__ import annotations

import types


def shard_bounds(V: int, g: int, rank: int):
    """Contiguous, as-even-as-possible vocab rows [v0, v1) of `rank` among `g` shards."""
    if not (0 <= rank < g):
        raise ValueError(f"rank {rank} out of range for {g} shards")
    return V * rank // g, V * (rank + 1) // g


def cuda_ops():
    from . import lce
    return types.SimpleNamespace(shard_stats=lce.shard_stats, stats_combine=lce.stats_combine, lce_bwd=lce.lce_bwd,
                                 dx_finalize=lce.dx_finalize)


class VocabShardedLCE:
    """Fused LCE with the LM head split by vocabulary rows across the ranks of `group`."""

    def __init__(self, V_global: int, group=None, ops=None, budget_bytes: int = 0):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.g = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.V = V_global
        self.v0, self.v1 = shard_bounds(V_global, self.g, self.rank)
        self.ops = ops or cuda_ops()
        self.budget = budget_bytes
        self._bufs = {}

    def _buf(self, key, shape, dtype, device):
        import torch
        b = self._bufs.get(key)
        if b is None or b.shape != shape or b.dtype != dtype or b.device != device:
            b = torch.empty(shape, dtype=dtype, device=device)
            self._bufs[key] = b
        return b

    def forward_backward(self, X, W_local, t, ignore_index: int = -100, reduction: str = "mean",
                         scale: float = 1.0, workspace=None, dW_out=None, dX_out=None):
        """Returns (loss, dX bf16 [N, H] (replicated), dW_local [V_k, H])."""
        import torch
        N, H = X.shape
        V_l = self.v1 - self.v0
        if W_local.shape[0] != V_l:
            raise ValueError(f"rank {self.rank} expects {V_l} vocab rows, got {W_local.shape[0]}")
        st = self.ops.shard_stats(X, W_local, t, self.v0, ignore_index=ignore_index, workspace=workspace,
                                  budget_bytes=self.budget)
        allst = self._buf("stats", (self.g, N, 4), st.dtype, st.device)
        self.dist.all_gather_into_tensor(allst.view(self.g * N, 4), st.contiguous(), group=self.group)
        loss, rs = self.ops.stats_combine(allst, t, self.v0, V_l, self.V, ignore_index=ignore_index,
                                          reduction=reduction, scale=scale, workspace=workspace)
        acc_dtype = torch.float64 if X.dtype == torch.float64 else torch.float32  # fp32 partials on the GPU path
        dx32 = self._buf("dx32", (N, H), acc_dtype, X.device)
        dW = dW_out if dW_out is not None else torch.empty_like(W_local)
        self.ops.lce_bwd(X, W_local, t, rs, 1.0, dhidden_fp32=True, workspace=workspace, budget_bytes=self.budget,
                         out=(dx32, dW))
        self.dist.all_reduce(dx32, group=self.group)
        dX = self.ops.dx_finalize(dx32, rs, out=dX_out)
        return loss, dX, dW
