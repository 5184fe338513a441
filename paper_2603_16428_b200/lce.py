"""Python API of the fused linear-cross-entropy hot path (thin layer over libslf_lce.so).

Every step of the path runs in the library's CUDA kernels; this module only checks dtypes,
allocates outputs / workspace with torch and passes pointers and the current stream.
Semantics: include/slf_lce.h and DESIGN.md (§3.3 fused LinearCrossEntropy).
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import REDUCTIONS, SCHEDULES, check, lib

ROWSTAT_BYTES = 16
SHARDSTAT_BYTES = 16


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _prep(hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor):
    if not (hidden.is_cuda and weight.is_cuda and targets.is_cuda):
        raise ValueError("hidden, weight and targets must be CUDA tensors (no CPU path)")
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise TypeError("hidden and weight must be bfloat16")
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
        raise ValueError(f"shape mismatch: hidden {tuple(hidden.shape)} weight {tuple(weight.shape)}")
    hidden = hidden.contiguous()
    weight = weight.contiguous()
    targets = targets.reshape(-1)
    if targets.dtype != torch.int32:
        targets = targets.to(torch.int32)
    targets = targets.contiguous()
    if targets.numel() != hidden.shape[0]:
        raise ValueError("targets must have N entries")
    return hidden, weight, targets


def workspace_bytes(N: int, H: int, V: int, schedule: str = "auto", budget_bytes: int = 0) -> int:
    return int(lib().slf_lce_workspace_bytes(N, H, V, SCHEDULES[schedule], budget_bytes))


def plan_describe(N: int, H: int, V: int, schedule: str = "auto", budget_bytes: int = 0) -> str:
    buf = ctypes.create_string_buffer(512)
    check(lib().slf_lce_plan_describe(N, H, V, SCHEDULES[schedule], budget_bytes, buf, 512), "slf_lce_plan_describe")
    return buf.value.decode()


def alloc_workspace(N: int, H: int, V: int, device, schedule: str = "auto", budget_bytes: int = 0) -> torch.Tensor:
    nb = workspace_bytes(N, H, V, schedule, budget_bytes)
    if nb == 0:
        raise RuntimeError(f"no LCE plan fits the budget for N={N} H={H} V={V} budget={budget_bytes}")
    return torch.empty(nb, dtype=torch.uint8, device=device)


def lce_fwd_bwd(hidden, weight, targets, ignore_index: int = -100, reduction: str = "mean", scale: float = 1.0,
                need_dhidden: bool = True, need_dweight: bool = True, budget_bytes: int = 0, workspace=None,
                out=None, schedule: str = "auto", accumulate_dw: bool = False, group=None, V_global: int = None):
    """Fused LCE forward + backward.  Returns (loss fp32, dhidden bf16 | None, dweight bf16 | None).

    ``out`` may be a (loss, dhidden, dweight) triple of preallocated tensors to write into;
    ``accumulate_dw`` adds dL/dW into the given dweight (gradient accumulation) instead of
    overwriting it.  With ``group`` (a torch.distributed process group, one rank per GPU) the LM
    head is vocab-sharded (SURVEY §8(b) "Python"): ``weight`` is this rank's rows
    [V_global*k/g, V_global*(k+1)/g) and the call is slf_lce_fwd_bwd_sharded over the library's
    own NCCL communicator for the group (created once and cached); the loss and dhidden are the
    global ones on every rank, dweight this rank's rows.
    """
    if group is not None:
        if V_global is None:
            raise ValueError("a vocab-sharded call (group=...) needs V_global")
        if accumulate_dw or schedule == "R":
            raise NotImplementedError("the sharded call runs schedule S and overwrites dweight")
        return lce_fwd_bwd_sharded(hidden, weight, targets, V_global, comm_for_group(group, hidden.device),
                                   ignore_index, reduction, scale, budget_bytes, workspace, out, need_dhidden,
                                   need_dweight)
    hidden, weight, targets = _prep(hidden, weight, targets)
    N, H = hidden.shape
    V = weight.shape[0]
    dev = hidden.device
    red = REDUCTIONS[reduction]
    if out is not None:
        loss, dX, dW = out
    else:
        loss = torch.empty(N if reduction == "none" else 1, dtype=torch.float32, device=dev)
        dX = torch.empty_like(hidden) if need_dhidden else None
        dW = torch.empty_like(weight) if need_dweight else None
    if workspace is None:
        workspace = alloc_workspace(N, H, V, dev, schedule, budget_bytes)
    if accumulate_dw and (out is None or dW is None):
        raise ValueError("accumulate_dw needs the dweight buffer to accumulate into (out=(loss, dX, dW))")
    check(lib().slf_lce_fwd_bwd_ex(hidden.data_ptr(), weight.data_ptr(), targets.data_ptr(), N, H, V, ignore_index,
                                   red, float(scale), loss.data_ptr(), _ptr(dX), _ptr(dW), workspace.data_ptr(),
                                   workspace.numel(), SCHEDULES[schedule], budget_bytes, int(bool(accumulate_dw)),
                                   _stream_ptr(dev)), "slf_lce_fwd_bwd_ex")
    return (loss if reduction == "none" else loss[0]), dX, dW


class HostStaging:
    """Device staging buffers for lce_fwd_bwd_host (hidden [N, H] bf16, targets [N] int32, loss)."""

    def __init__(self, N: int, H: int, device, reduction: str = "mean"):
        self.hidden = torch.empty(N, H, dtype=torch.bfloat16, device=device)
        self.targets = torch.empty(N, dtype=torch.int32, device=device)
        self.loss = torch.empty(N if reduction == "none" else 1, dtype=torch.float32, device=device)


def lce_fwd_bwd_host(hidden_host, weight, targets_host, ignore_index: int = -100, reduction: str = "mean",
                     scale: float = 1.0, dX=None, dW=None, loss_host=None, staging: HostStaging = None,
                     workspace=None, budget_bytes: int = 0, schedule: str = "auto", accumulate_dw: bool = False):
    """The fused call with HOST hidden states / targets / loss (slf_lce_fwd_bwd_host): the row chunks
    of hidden are copied on an internal stream while earlier chunks compute.  hidden_host: CPU bf16
    [N, H] (pin it for overlap), targets_host: CPU int32 [N].  Returns (loss_host (valid after the
    current stream synchronises), dX, dW) — gradients stay on the device."""
    if hidden_host.is_cuda or targets_host.is_cuda:
        raise TypeError("hidden_host / targets_host must be CPU tensors")
    if hidden_host.dtype != torch.bfloat16 or targets_host.dtype != torch.int32:
        raise TypeError("hidden_host must be bf16, targets_host int32")
    if not (hidden_host.is_contiguous() and targets_host.is_contiguous()):
        raise ValueError("host tensors must be contiguous")
    N, H = hidden_host.shape
    V = weight.shape[0]
    dev = weight.device
    n_loss = N if reduction == "none" else 1
    if staging is None:
        staging = HostStaging(N, H, dev, reduction)
    elif (tuple(staging.hidden.shape) != (N, H) or staging.targets.numel() < N or staging.loss.numel() < n_loss
          or staging.hidden.device != dev):
        raise ValueError(f"staging buffers (hidden {tuple(staging.hidden.shape)}, targets {staging.targets.numel()}, "
                         f"loss {staging.loss.numel()}) do not fit N={N} H={H} reduction={reduction!r}")
    if loss_host is None:
        loss_host = torch.empty(n_loss, dtype=torch.float32).pin_memory()
    elif loss_host.is_cuda or loss_host.dtype != torch.float32 or loss_host.numel() < n_loss:
        raise ValueError(f"loss_host must be a CPU float32 tensor of >= {n_loss} elements")
    if dX is None:
        dX = torch.empty(N, H, dtype=torch.bfloat16, device=dev)
    if dW is None and not accumulate_dw:
        dW = torch.empty_like(weight)
    if workspace is None:
        workspace = alloc_workspace(N, H, V, dev, schedule, budget_bytes)
    check(lib().slf_lce_fwd_bwd_host(hidden_host.data_ptr(), weight.data_ptr(), targets_host.data_ptr(), N, H, V,
                                     ignore_index, REDUCTIONS[reduction], float(scale), loss_host.data_ptr(),
                                     _ptr(dX), _ptr(dW), staging.hidden.data_ptr(), staging.targets.data_ptr(),
                                     staging.loss.data_ptr(), workspace.data_ptr(), workspace.numel(),
                                     SCHEDULES[schedule], budget_bytes, int(bool(accumulate_dw)), _stream_ptr(dev)),
          "slf_lce_fwd_bwd_host")
    return loss_host, dX, dW


def lce_fwd(hidden, weight, targets, ignore_index: int = -100, reduction: str = "mean", scale: float = 1.0,
            budget_bytes: int = 0, workspace=None):
    """Forward half (schedule R split).  Returns (loss, rowstat [N, 16 bytes as uint8])."""
    hidden, weight, targets = _prep(hidden, weight, targets)
    N, H = hidden.shape
    V = weight.shape[0]
    dev = hidden.device
    loss = torch.empty(N if reduction == "none" else 1, dtype=torch.float32, device=dev)
    rowstat = torch.empty(N, ROWSTAT_BYTES, dtype=torch.uint8, device=dev)
    if workspace is None:
        workspace = alloc_workspace(N, H, V, dev, budget_bytes=budget_bytes)
    check(lib().slf_lce_fwd(hidden.data_ptr(), weight.data_ptr(), targets.data_ptr(), N, H, V, ignore_index,
                            REDUCTIONS[reduction], float(scale), loss.data_ptr(), rowstat.data_ptr(),
                            workspace.data_ptr(), workspace.numel(), budget_bytes, _stream_ptr(dev)), "slf_lce_fwd")
    return (loss if reduction == "none" else loss[0]), rowstat


def lce_bwd(hidden, weight, targets, rowstat, grad_scale: float = 1.0, need_dhidden: bool = True,
            need_dweight: bool = True, dhidden_fp32: bool = False, budget_bytes: int = 0, workspace=None,
            out=None):
    """Backward half: recompute logits per tile, G -> dhidden, dweight.  grad_scale = upstream grad.

    ``out`` may be a preallocated (dhidden, dweight) pair (either may be None to skip it)."""
    hidden, weight, targets = _prep(hidden, weight, targets)
    N, H = hidden.shape
    V = weight.shape[0]
    dev = hidden.device
    if out is not None:
        dX, dW = out
    else:
        dX = None
        if need_dhidden:
            dX = torch.empty(N, H, dtype=torch.float32 if dhidden_fp32 else torch.bfloat16, device=dev)
        dW = torch.empty_like(weight) if need_dweight else None
    if workspace is None:
        workspace = alloc_workspace(N, H, V, dev, budget_bytes=budget_bytes)
    check(lib().slf_lce_bwd(hidden.data_ptr(), weight.data_ptr(), targets.data_ptr(), rowstat.data_ptr(), N, H, V,
                            float(grad_scale), _ptr(dX), int(dhidden_fp32), _ptr(dW), workspace.data_ptr(),
                            workspace.numel(), budget_bytes, _stream_ptr(dev)), "slf_lce_bwd")
    return dX, dW


def shard_stats(hidden, weight_shard, targets, vocab_start: int, ignore_index: int = -100, budget_bytes: int = 0,
                workspace=None):
    """This vocab shard's per-row (m, s, z_t, hit) as a float32 [N, 4] tensor."""
    hidden, weight_shard, targets = _prep(hidden, weight_shard, targets)
    N, H = hidden.shape
    V_l = weight_shard.shape[0]
    dev = hidden.device
    st = torch.empty(N, 4, dtype=torch.float32, device=dev)
    if workspace is None:
        workspace = alloc_workspace(N, H, V_l, dev, budget_bytes=budget_bytes)
    check(lib().slf_lce_fwd_shard_stats(hidden.data_ptr(), weight_shard.data_ptr(), targets.data_ptr(), N, H, V_l,
                                        vocab_start, ignore_index, st.data_ptr(), workspace.data_ptr(),
                                        workspace.numel(), budget_bytes, _stream_ptr(dev)), "slf_lce_fwd_shard_stats")
    return st


def stats_combine(stats, targets, vocab_start: int, V_local: int, V_global: int, ignore_index: int = -100,
                  reduction: str = "mean", scale: float = 1.0, workspace=None):
    """Merge [g, N, 4] shard statistics (shard order) into (loss, this shard's rowstat)."""
    if stats.dtype != torch.float32 or stats.dim() != 3 or stats.shape[2] != 4:
        raise ValueError("stats must be float32 [g, N, 4]")
    stats = stats.contiguous()
    g, N, _ = stats.shape
    targets = targets.reshape(-1).to(torch.int32).contiguous()
    dev = stats.device
    loss = torch.empty(N if reduction == "none" else 1, dtype=torch.float32, device=dev)
    rowstat = torch.empty(N, ROWSTAT_BYTES, dtype=torch.uint8, device=dev)
    if workspace is None:
        workspace = torch.empty(64 * 1024, dtype=torch.uint8, device=dev)
    check(lib().slf_lce_stats_combine(stats.data_ptr(), g, targets.data_ptr(), N, vocab_start, V_local, V_global,
                                      ignore_index, REDUCTIONS[reduction], float(scale), loss.data_ptr(),
                                      rowstat.data_ptr(), workspace.data_ptr(), workspace.numel(), _stream_ptr(dev)),
          "slf_lce_stats_combine")
    return (loss if reduction == "none" else loss[0]), rowstat


def status(workspace, device=None):
    """(bad_targets, n_valid) of the last call that used this workspace (synchronises the stream)."""
    bad = ctypes.c_int32(0)
    nv = ctypes.c_int64(0)
    check(lib().slf_lce_status(workspace.data_ptr(), _stream_ptr(device or workspace.device), ctypes.byref(bad),
                               ctypes.byref(nv)), "slf_lce_status")
    return bad.value, nv.value


def target_csr(targets, V_local: int, vocab_start: int = 0, ignore_index: int = -100):
    """Target CSR of a vocabulary shard (slf_target_csr): returns (offsets [V_local + 2] int32,
    token_idx [N] int32) on the targets' device; see include/slf_lce.h."""
    if not targets.is_cuda or targets.dtype != torch.int32 or not targets.is_contiguous():
        raise TypeError("targets must be a contiguous CUDA int32 tensor")
    N = targets.numel()
    dev = targets.device
    offsets = torch.empty(V_local + 2, dtype=torch.int32, device=dev)
    idx = torch.empty(N, dtype=torch.int32, device=dev)
    nb = lib().slf_target_csr_scratch_bytes(N, V_local)
    scratch = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev)
    check(lib().slf_target_csr(targets.data_ptr(), N, ignore_index, vocab_start, V_local, offsets.data_ptr(),
                               idx.data_ptr(), scratch.data_ptr(), scratch.numel(), _stream_ptr(dev)), "slf_target_csr")
    return offsets, idx


def dx_finalize(dx32, rowstat, out=None):
    """bf16 dhidden from the fp32 sum of shard partials (ignored rows -> +0.0)."""
    N, H = dx32.shape
    if out is None:
        out = torch.empty(N, H, dtype=torch.bfloat16, device=dx32.device)
    check(lib().slf_lce_dx_finalize(dx32.data_ptr(), rowstat.data_ptr(), out.data_ptr(), N, H,
                                    _stream_ptr(dx32.device)), "slf_lce_dx_finalize")
    return out


# ---- schedule S split for vocab shards (include/slf_lce.h) ---------------------------------------
def s_plan(N: int, H: int, V_local: int, budget_bytes: int = 0):
    """(chunk_rows, n_chunks) of the schedule-S plan."""
    c, n = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib().slf_lce_s_plan(N, H, V_local, budget_bytes, ctypes.byref(c), ctypes.byref(n)), "slf_lce_s_plan")
    return c.value, n.value


class SShard:
    """One step of schedule S on this rank's vocab shard, driven chunk by chunk (the caller does the
    collectives between the calls; see paper_2603_16428_b200.sharded)."""

    def __init__(self, hidden, weight_shard, targets, vocab_start: int, V_global: int, ignore_index: int = -100,
                 reduction: str = "mean", scale: float = 1.0, budget_bytes: int = 0, workspace=None):
        self.X, self.W, self.t = _prep(hidden, weight_shard, targets)
        self.N, self.H = self.X.shape
        self.V_l = self.W.shape[0]
        self.vs, self.V = vocab_start, V_global
        self.ign, self.red, self.scale = ignore_index, REDUCTIONS[reduction], float(scale)
        self.budget = budget_bytes
        self.C, self.n_chunks = s_plan(self.N, self.H, self.V_l, budget_bytes)
        dev = self.X.device
        self.ws = workspace if workspace is not None else alloc_workspace(self.N, self.H, self.V_l, dev, "S",
                                                                           budget_bytes)
        self.stream = _stream_ptr(dev)

    def rows(self, ch: int):
        r0 = ch * self.C
        return r0, min(self.C, self.N - r0)

    def begin(self, need_dweight: bool = True):
        check(lib().slf_lce_s_begin(self.t.data_ptr(), self.N, self.H, self.V_l, self.vs, self.V, self.ign,
                                    int(need_dweight), self.ws.data_ptr(), self.ws.numel(), self.budget, self.stream),
              "slf_lce_s_begin")

    def chunk_stats(self, ch: int, out=None):
        r0, rows = self.rows(ch)
        st = out if out is not None else torch.empty(rows, 4, dtype=torch.float32, device=self.X.device)
        check(lib().slf_lce_s_chunk_stats(self.X.data_ptr(), self.W.data_ptr(), self.t.data_ptr(), self.N, self.H,
                                          self.V_l, self.vs, self.V, self.ign, ch, st.data_ptr(), self.ws.data_ptr(),
                                          self.ws.numel(), self.budget, self.stream), "slf_lce_s_chunk_stats")
        return st

    def chunk_bwd(self, ch: int, stats, dX_chunk=None, dhidden_fp32: bool = True, dW=None, loss_rows=None):
        """stats: float32 [g, rows, 4] (rank order)."""
        g = stats.shape[0]
        check(lib().slf_lce_s_chunk_bwd(self.X.data_ptr(), self.W.data_ptr(), self.t.data_ptr(), self.N, self.H,
                                        self.V_l, self.vs, self.V, self.ign, self.red, self.scale, ch,
                                        stats.data_ptr(), g, _ptr(loss_rows), _ptr(dX_chunk), int(dhidden_fp32),
                                        _ptr(dW), self.ws.data_ptr(), self.ws.numel(), self.budget, self.stream),
              "slf_lce_s_chunk_bwd")

    def end(self, loss_out=None, dW=None):
        check(lib().slf_lce_s_end(self.X.data_ptr(), self.N, self.H, self.V_l, self.red, self.scale, _ptr(loss_out),
                                  _ptr(dW), self.ws.data_ptr(), self.ws.numel(), self.budget, self.stream),
              "slf_lce_s_end")

    def rowstat(self):
        """Device address of the step's RowStat array [N] (inside the workspace)."""
        p = ctypes.c_void_p(0)
        check(lib().slf_lce_s_rowstat(self.N, self.H, self.V_l, self.budget, self.ws.data_ptr(), ctypes.byref(p)),
              "slf_lce_s_rowstat")
        return p.value


def rmsnorm_fwd(x, g, eps: float = 1e-5):
    """Final RMSNorm: (y bf16 [N, H], rstd fp32 [N])."""
    if x.dtype != torch.bfloat16 or g.dtype != torch.bfloat16 or not x.is_cuda:
        raise TypeError("x and g must be bf16 CUDA tensors")
    x = x.contiguous()
    N, H = x.shape
    y = torch.empty_like(x)
    rstd = torch.empty(N, dtype=torch.float32, device=x.device)
    check(lib().slf_rmsnorm_fwd(x.data_ptr(), g.contiguous().data_ptr(), N, H, float(eps), y.data_ptr(),
                                rstd.data_ptr(), _stream_ptr(x.device)), "slf_rmsnorm_fwd")
    return y, rstd


def rmsnorm_workspace_bytes(N: int, H: int) -> int:
    return int(lib().slf_rmsnorm_workspace_bytes(N, H))


def rmsnorm_bwd(x, g, rstd, dy, dx=None, workspace=None, dg=None):
    """RMSNorm VJP: (dx bf16 [N, H], dg fp32 [H]).  dx may be dy (in place).  `workspace` (uint8,
    >= rmsnorm_workspace_bytes(N, H)) avoids an allocation per call."""
    x = x.contiguous()
    N, H = x.shape
    dx = dx if dx is not None else torch.empty_like(x)
    dg = dg if dg is not None else torch.empty(H, dtype=torch.float32, device=x.device)
    ws = workspace if workspace is not None else torch.empty(rmsnorm_workspace_bytes(N, H), dtype=torch.uint8,
                                                            device=x.device)
    check(lib().slf_rmsnorm_bwd(x.data_ptr(), g.contiguous().data_ptr(), rstd.data_ptr(), dy.data_ptr(), N, H,
                                dx.data_ptr(), dg.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(x.device)),
          "slf_rmsnorm_bwd")
    return dx, dg


def rmsnorm_lce_workspace_bytes(N: int, H: int, V: int, budget_bytes: int = 0) -> int:
    return int(lib().slf_rmsnorm_lce_workspace_bytes(N, H, V, budget_bytes))


def rmsnorm_lce_plan_describe(N: int, H: int, V: int, budget_bytes: int = 0) -> str:
    buf = ctypes.create_string_buffer(512)
    check(lib().slf_rmsnorm_lce_plan_describe(N, H, V, budget_bytes, buf, 512), "slf_rmsnorm_lce_plan_describe")
    return buf.value.decode()


def rmsnorm_lce_fwd_bwd(x, g, weight, targets, eps: float = 1e-5, ignore_index: int = -100,
                        reduction: str = "mean", scale: float = 1.0, budget_bytes: int = 0, workspace=None,
                        schedule: str = "auto", fused: bool = True, out=None):
    """Final RMSNorm + fused LCE, forward and backward: (loss, dx (pre-norm), dg fp32, dW).

    fused (default; schedule auto/S): one library call, slf_rmsnorm_lce_fwd_bwd — y only ever exists
    for one row chunk.  fused=False or schedule R: the composition rmsnorm_fwd -> lce_fwd_bwd ->
    rmsnorm_bwd (y [N, H] materialised; the LCE's dhidden fed through the VJP in place)."""
    if fused and schedule in ("auto", "S"):
        x, weight, targets = _prep(x, weight, targets)
        N, H = x.shape
        V = weight.shape[0]
        dev = x.device
        if out is not None:
            loss, dx, dg, dW = out
        else:
            loss = torch.empty(N if reduction == "none" else 1, dtype=torch.float32, device=dev)
            dx = torch.empty_like(x)
            dg = torch.empty(H, dtype=torch.float32, device=dev)
            dW = torch.empty_like(weight)
        if workspace is None:
            nb = rmsnorm_lce_workspace_bytes(N, H, V, budget_bytes)
            if nb == 0:
                raise RuntimeError(f"no fused RMSNorm+LCE plan fits N={N} H={H} V={V} budget={budget_bytes}")
            workspace = torch.empty(nb, dtype=torch.uint8, device=dev)
        check(lib().slf_rmsnorm_lce_fwd_bwd(x.data_ptr(), g.contiguous().data_ptr(), float(eps), weight.data_ptr(),
                                            targets.data_ptr(), N, H, V, ignore_index, REDUCTIONS[reduction],
                                            float(scale), loss.data_ptr(), dx.data_ptr(), dg.data_ptr(),
                                            dW.data_ptr(), workspace.data_ptr(), workspace.numel(), budget_bytes,
                                            _stream_ptr(dev)), "slf_rmsnorm_lce_fwd_bwd")
        return (loss if reduction == "none" else loss[0]), dx, dg, dW
    y, rstd = rmsnorm_fwd(x, g, eps)
    loss, dy, dW = lce_fwd_bwd(y, weight, targets, ignore_index, reduction, scale, budget_bytes=budget_bytes,
                               workspace=workspace, schedule=schedule)
    dx, dg = rmsnorm_bwd(x, g, rstd, dy, dx=dy)
    return loss, dx, dg, dW


def dx_finalize_ptr(dx32, rowstat_ptr: int, out):
    """dx_finalize with a raw RowStat device address (rows already offset by the caller)."""
    N, H = dx32.shape
    check(lib().slf_lce_dx_finalize(dx32.data_ptr(), rowstat_ptr, out.data_ptr(), N, H, _stream_ptr(dx32.device)),
          "slf_lce_dx_finalize")
    return out


# ---- vocab-sharded call with the collectives inside the library (include/slf_lce.h "Comm") ---------
def comm_unique_id() -> bytes:
    """128-byte NCCL bootstrap id (rank 0 creates it; ship it to every rank)."""
    buf = ctypes.create_string_buffer(128)
    check(lib().slf_comm_get_unique_id(buf), "slf_comm_get_unique_id")
    return buf.raw


class Comm:
    """slf_comm handle: one process = one GPU = one rank of the vocab-sharded LM head."""

    def __init__(self, handle, rank: int, world: int, keep=None):
        self.handle, self.rank, self.world = handle, rank, world
        self._keep = keep  # ctypes callbacks must outlive the handle
        self.p2p_mode = 0

    @classmethod
    def nccl(cls, unique_id: bytes, rank: int, world: int, device: int):
        h = ctypes.c_void_p(0)
        check(lib().slf_comm_init(ctypes.byref(h), ctypes.create_string_buffer(bytes(unique_id), 128), rank, world,
                                  device), "slf_comm_init")
        return cls(h.value, rank, world)

    @classmethod
    def from_process_group(cls, group=None, device=None):
        """NCCL communicator over the ranks of a torch.distributed group (bootstrap id broadcast
        from the group's first rank; torch is plumbing here, the collectives run in the library)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        dev = torch.cuda.current_device() if device is None else int(device)
        return cls.nccl(obj[0], rank, world, dev)

    @classmethod
    def callbacks(cls, rank: int, world: int, allgather, allreduce_f32):
        """Caller transport: allgather(send_ptr, recv_ptr, bytes_per_rank, stream_ptr) and
        allreduce_f32(buf_ptr, count, stream_ptr), device addresses; run synchronously."""
        from ._lib import ALLGATHER_FN, ALLREDUCE_FN

        def ag(send, recv, nbytes, stream, user):
            try:
                allgather(send, recv, nbytes, stream)
                return 0
            except Exception as e:  # noqa: BLE001 — reported as SLF_ERR_COMM
                print(f"allgather callback failed: {e!r}")
                return 1

        def ar(buf, count, stream, user):
            try:
                allreduce_f32(buf, count, stream)
                return 0
            except Exception as e:  # noqa: BLE001
                print(f"allreduce callback failed: {e!r}")
                return 1

        fa, fr = ALLGATHER_FN(ag), ALLREDUCE_FN(ar)
        h = ctypes.c_void_p(0)
        check(lib().slf_comm_init_callbacks(ctypes.byref(h), rank, world, fa, fr, None), "slf_comm_init_callbacks")
        return cls(h.value, rank, world, keep=(fa, fr))

    def set_p2p(self, enable=True):
        """P2P exchanges over CUDA IPC (slf_comm_set_p2p): True / 1 the per-chunk statistics
        all-gather, 2 the dX exchange kernel, 3 both; False / 0 off."""
        check(lib().slf_comm_set_p2p(self.handle, int(enable)), "slf_comm_set_p2p")
        self.p2p_mode = int(enable)
        return self

    def p2p_timeouts(self) -> int:
        v = ctypes.c_int32(0)
        check(lib().slf_comm_status(self.handle, ctypes.byref(v)), "slf_comm_status")
        return v.value

    def close(self):
        if self.handle:
            check(lib().slf_comm_destroy(self.handle), "slf_comm_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass


_COMMS = {}


def comm_for_group(group, device):
    """The library communicator of a torch.distributed group on `device` (created on first use)."""
    import torch.distributed as dist
    key = (id(group), str(device))
    c = _COMMS.get(key)
    if c is None or c.handle is None:
        c = Comm.from_process_group(None if group is dist.group.WORLD else group, device=device.index)
        _COMMS[key] = c
    return c


def shard_bounds_native(V_global: int, world: int, rank: int):
    v0, vl = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib().slf_shard_bounds(V_global, world, rank, ctypes.byref(v0), ctypes.byref(vl)), "slf_shard_bounds")
    return v0.value, v0.value + vl.value


def sharded_workspace_bytes(N: int, H: int, V_global: int, world: int, rank: int, budget_bytes: int = 0) -> int:
    return int(lib().slf_lce_sharded_workspace_bytes(N, H, V_global, world, rank, budget_bytes))


def sharded_plan_describe(N: int, H: int, V_global: int, world: int, rank: int, budget_bytes: int = 0) -> str:
    buf = ctypes.create_string_buffer(512)
    check(lib().slf_lce_sharded_plan_describe(N, H, V_global, world, rank, budget_bytes, buf, 512),
          "slf_lce_sharded_plan_describe")
    return buf.value.decode()


def sharded_chunk_table(N: int, H: int, V_global: int, world: int, rank: int, budget_bytes: int = 0):
    """The sharded call's row chunks (slf_lce_sharded_chunk_table): a list of dicts with r0, rows,
    ext, part_off (bytes into dhidden; -1 workspace stash tail, -2 workspace region), xt_lim, ld."""
    n = ctypes.c_int64(0)
    check(lib().slf_lce_sharded_chunk_table(N, H, V_global, world, rank, budget_bytes, None, 0, ctypes.byref(n)),
          "slf_lce_sharded_chunk_table")
    buf = (ctypes.c_int64 * (6 * max(1, n.value)))()
    check(lib().slf_lce_sharded_chunk_table(N, H, V_global, world, rank, budget_bytes, buf, n.value, ctypes.byref(n)),
          "slf_lce_sharded_chunk_table")
    keys = ("r0", "rows", "ext", "part_off", "xt_lim", "ld")
    return [dict(zip(keys, buf[6 * i:6 * i + 6])) for i in range(n.value)]


def lce_fwd_bwd_sharded(hidden, weight_shard, targets, V_global: int, comm: Comm, ignore_index: int = -100,
                        reduction: str = "mean", scale: float = 1.0, budget_bytes: int = 0, workspace=None,
                        out=None, need_dhidden: bool = True, need_dweight: bool = True, check_p2p: bool = True):
    """Vocab-sharded fused LCE on this rank (slf_lce_fwd_bwd_sharded): every rank passes the same
    hidden / targets and its own W rows; returns (global loss, full dhidden, this rank's dW rows).

    With P2P exchanges enabled on ``comm`` and ``check_p2p`` (default), the call synchronises and
    raises if a P2P wait timed out (a peer more than ~30 s late: the results would be stale).  With
    ``check_p2p=False`` the library still poisons that call's loss with NaN and fails the next call."""
    hidden, weight_shard, targets = _prep(hidden, weight_shard, targets)
    N, H = hidden.shape
    v0, v1 = shard_bounds_native(V_global, comm.world, comm.rank)
    if weight_shard.shape[0] != v1 - v0:
        raise ValueError(f"rank {comm.rank} expects {v1 - v0} vocab rows, got {weight_shard.shape[0]}")
    dev = hidden.device
    if out is not None:
        loss, dX, dW = out
    else:
        loss = torch.empty(N if reduction == "none" else 1, dtype=torch.float32, device=dev)
        dX = torch.empty_like(hidden) if need_dhidden else None
        dW = torch.empty_like(weight_shard) if need_dweight else None
    if workspace is None:
        nb = sharded_workspace_bytes(N, H, V_global, comm.world, comm.rank, budget_bytes)
        if nb == 0:
            raise RuntimeError(f"no sharded plan fits N={N} H={H} V={V_global} world={comm.world}")
        workspace = torch.empty(nb, dtype=torch.uint8, device=dev)
    check(lib().slf_lce_fwd_bwd_sharded(hidden.data_ptr(), weight_shard.data_ptr(), targets.data_ptr(), N, H,
                                        V_global, ignore_index, REDUCTIONS[reduction], float(scale), loss.data_ptr(),
                                        _ptr(dX), _ptr(dW), workspace.data_ptr(), workspace.numel(), budget_bytes,
                                        comm.handle, _stream_ptr(dev)), "slf_lce_fwd_bwd_sharded")
    if check_p2p and comm.p2p_mode and comm.p2p_timeouts():
        raise RuntimeError(f"rank {comm.rank}: a P2P exchange wait timed out; this step's results are invalid")
    return (loss if reduction == "none" else loss[0]), dX, dW



def lce_fwd_bwd_dp(hidden, weight, targets, comm: Comm, ignore_index: int = -100, reduction: str = "mean",
                   scale: float = 1.0, sync_dweight: bool = False, budget_bytes: int = 0, workspace=None, out=None,
                   schedule: str = "auto"):
    """Data-parallel fused LCE on this rank (slf_lce_fwd_bwd_dp): this rank's tokens, the full W;
    returns (global loss, local dhidden, dW partial — or the all-reduced dW with sync_dweight)."""
    hidden, weight, targets = _prep(hidden, weight, targets)
    N, H = hidden.shape
    V = weight.shape[0]
    dev = hidden.device
    if out is not None:
        loss, dX, dW = out
    else:
        loss = torch.empty(N if reduction == "none" else 1, dtype=torch.float32, device=dev)
        dX = torch.empty_like(hidden)
        dW = torch.empty_like(weight)
    if workspace is None:
        workspace = alloc_workspace(N, H, V, dev, schedule, budget_bytes)
    check(lib().slf_lce_fwd_bwd_dp(hidden.data_ptr(), weight.data_ptr(), targets.data_ptr(), N, H, V, ignore_index,
                                   REDUCTIONS[reduction], float(scale), loss.data_ptr(), _ptr(dX), _ptr(dW),
                                   workspace.data_ptr(), workspace.numel(), SCHEDULES[schedule], budget_bytes,
                                   int(bool(sync_dweight)), comm.handle, _stream_ptr(dev)), "slf_lce_fwd_bwd_dp")
    return (loss if reduction == "none" else loss[0]), dX, dW

class Profile:
    """Context manager over slf_profile_begin/end: per-kernel-kind device ms, launches, FLOPs, bytes."""

    def __enter__(self):
        check(lib().slf_profile_begin(), "slf_profile_begin")
        return self

    def __exit__(self, *exc):
        from ._lib import PROF_KINDS
        n = len(PROF_KINDS)
        ms = (ctypes.c_double * n)()
        la = (ctypes.c_int64 * n)()
        fl = (ctypes.c_double * n)()
        by = (ctypes.c_double * n)()
        check(lib().slf_profile_end(ms, la, fl, by), "slf_profile_end")
        self.kinds = {k: dict(ms=ms[i], launches=la[i], flops=fl[i], bytes=by[i])
                      for i, k in enumerate(PROF_KINDS) if la[i]}
        return False


def debug_gemm(A, B, a_mn: bool, b_mn: bool, M: int, N: int, K: int):
    """D[M, N] fp32 = A * B through the tcgen05 core (see slf_debug_gemm)."""
    D = torch.empty(M, N, dtype=torch.float32, device=A.device)
    check(lib().slf_debug_gemm(A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, int(a_mn), int(b_mn),
                               _stream_ptr(A.device)), "slf_debug_gemm")
    return D


def scale_(t, s: float):
    """In-place t *= s for a contiguous bf16 CUDA tensor (library kernel)."""
    if s == 1.0 or t is None:
        return t
    check(lib().slf_scale_bf16(t.data_ptr(), t.numel(), float(s), _stream_ptr(t.device)), "slf_scale_bf16")
    return t


def scale_dev_(t, s_dev):
    """In-place t *= s_dev[0] (a CUDA fp32 scalar tensor, read on the device); no-op pass for 1."""
    if t is None:
        return t
    s_dev = s_dev.detach().reshape(-1).to(torch.float32).contiguous()
    check(lib().slf_scale_bf16_dev(t.data_ptr(), t.numel(), s_dev.data_ptr(), _stream_ptr(t.device)),
          "slf_scale_bf16_dev")
    return t


def rowstat_scale(rowstat, grad, per_row: bool):
    """RowStat copy with coef *= grad (scalar or per row), on the device (slf_rowstat_scale)."""
    N = rowstat.numel() // 16
    grad = grad.detach().reshape(-1).to(torch.float32).contiguous()
    out = torch.empty_like(rowstat)
    check(lib().slf_rowstat_scale(rowstat.data_ptr(), grad.data_ptr(), int(per_row), N, out.data_ptr(),
                                  _stream_ptr(rowstat.device)), "slf_rowstat_scale")
    return out


class LCEFunctionFused(torch.autograd.Function):
    """autograd wrapper on the fused call (schedule S when it fits): the gradients are formed during
    the forward (no recompute) and scaled by grad_output in backward on the device (no host read; a
    no-op pass for grad_output == 1, otherwise one more bf16 rounding of the stored gradients —
    exact for powers of two; use LCEFunction to fold grad_output into the gradients' formation)."""

    @staticmethod
    def forward(ctx, hidden, weight, targets, ignore_index=-100, reduction="mean"):
        if reduction == "none":
            raise NotImplementedError("reduction='none' needs a per-row grad; use LCEFunction")
        loss, dX, dW = lce_fwd_bwd(hidden, weight, targets, ignore_index, reduction, 1.0,
                                   need_dhidden=ctx.needs_input_grad[0], need_dweight=ctx.needs_input_grad[1])
        ctx.grads = (dX, dW)
        return loss

    @staticmethod
    def backward(ctx, grad_out):
        dX, dW = ctx.grads
        ctx.grads = None
        return scale_dev_(dX, grad_out), scale_dev_(dW, grad_out), None, None, None


class LCEFunction(torch.autograd.Function):
    """autograd wrapper on the schedule-R split: forward keeps only the 16-byte RowStat per token."""

    @staticmethod
    def forward(ctx, hidden, weight, targets, ignore_index=-100, reduction="mean"):
        loss, rowstat = lce_fwd(hidden, weight, targets, ignore_index, reduction, 1.0)
        ctx.save_for_backward(hidden, weight, targets, rowstat)
        ctx.reduction = reduction
        return loss

    @staticmethod
    def backward(ctx, grad_out):
        hidden, weight, targets, rowstat = ctx.saved_tensors
        # grad_output folded into the per-row coefficients on the device (per row for 'none'): the
        # gradients are formed once, in fp32, already scaled; no host synchronisation.
        rs = rowstat_scale(rowstat, grad_out, per_row=ctx.reduction == "none")
        dX, dW = lce_bwd(hidden, weight, targets, rs, 1.0, ctx.needs_input_grad[0], ctx.needs_input_grad[1])
        return dX, dW, None, None, None
