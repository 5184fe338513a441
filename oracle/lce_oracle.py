"""Plain, slow, obviously-correct CPU oracle for the fused linear-cross-entropy.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2603_16428_b200``) never imports it, and it
shares no code with the CUDA library.

What it computes (§3.3 "Optimized Triton Kernels": the fused
LinearCrossEntropy kernel "fuses the projection and loss calculation, computing
gradients in small chunks to avoid materializing the full logits tensor ...
without sacrificing accuracy"; Fig. ``fig:lce`` caption, PAPER.md line 235,
compares against the "torch standard method").  The method therefore reaches
exactly the standard result, so this oracle is the plain definition of softmax
cross-entropy over the LM-head logits, written out in float64 and MATERIALISING
the logits (row block by row block; each block holds whole rows, so blocking
is exact):

    Z      = X W^T                                  (c1; [N, V])
    lse_i  = m_i + log sum_v exp(Z_iv - m_i),  m_i = max_v Z_iv        (c2)
    valid_i = (t_i != ignore_index)                 (reading R1)
    l_i    = valid_i ? lse_i - Z_{i,t_i} : 0
    loss   = sum_i l_i (SUM) | sum_i l_i / n_valid (MEAN; 0 if n_valid = 0, R2) | l (NONE)
    coef_i = scale * valid_i * (1/n_valid if MEAN else 1)          (c3; R3)
    G      = coef_i (softmax(Z_i) - e_{t_i})
    dX     = G W ,   dW = G^T X

Readings of the paper taken here are listed in DESIGN.md §Readings (R1-R9).
All inputs are float64 arrays; bf16 inputs are converted exactly by the caller
(``synth.bf16_bits_to_f64``).

Pinned by tests/test_oracle_pins.py (finite differences, the W = 0 closed form,
zero row sums, identical rows / V = 1, ignore masking, scale linearity,
SUM/MEAN ratio, torch float64 cross-entropy + autograd, a hand-derived golden
example, shard combination).
"""
from __future__ import annotations

import numpy as np

SUM, MEAN, NONE = "sum", "mean", "none"


def _coef(t: np.ndarray, ignore_index: int, reduction: str, scale: float):
    """coef_i of SURVEY §8(c) c3 / DESIGN.md R2-R3."""
    valid = t != ignore_index
    n_valid = int(valid.sum())
    if reduction == MEAN:
        per = (scale / n_valid) if n_valid > 0 else 0.0
    elif reduction in (SUM, NONE):
        per = scale
    else:
        raise ValueError(f"reduction must be sum|mean|none, got {reduction!r}")
    return valid, n_valid, np.where(valid, per, 0.0).astype(np.float64)


def rows(X: np.ndarray, W: np.ndarray, t: np.ndarray, coef: np.ndarray, ignore_index: int = -100):
    """Per-row loss, lse and dX for a set of rows, all V columns materialised.

    ``coef`` is given explicitly so a row slice of a large problem can be checked
    exactly (loss_i and dX_i depend only on row i once coef is fixed).
    Returns (l [n], lse [n], dX [n, H], G [n, V]).
    """
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    V = W.shape[0]
    Z = X @ W.T                                         # c1: the full logits rows
    m = Z.max(axis=1)                                   # c2: row max
    lse = m + np.log(np.exp(Z - m[:, None]).sum(axis=1))
    valid = t != ignore_index
    tt = np.where(valid, t, 0).astype(np.int64)
    z_t = Z[np.arange(Z.shape[0]), tt]
    loss_rows = np.where(valid, lse - z_t, 0.0)
    P = np.exp(Z - lse[:, None])                        # softmax(Z_i)
    onehot = np.zeros_like(P)
    onehot[np.arange(Z.shape[0])[valid], tt[valid]] = 1.0
    G = coef[:, None] * (P - onehot)                    # c3
    dX = G @ W
    return loss_rows, lse, dX, G


def lce(X, W, t, ignore_index: int = -100, reduction: str = MEAN, scale: float = 1.0,
        block_rows: int = 1024, need_grads: bool = True):
    """The plain definition (c1-c3) on the whole problem.

    Returns a dict: loss (scalar or [N]), dX [N, H], dW [V, H], lse [N], n_valid,
    bad_targets.  A valid target outside [0, V) is a data error (reading R4):
    loss becomes NaN and ``bad_targets`` counts them; gradients are not formed.
    """
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    t = np.asarray(t).astype(np.int64)
    N, H = X.shape
    V = W.shape[0]
    valid, n_valid, coef = _coef(t, ignore_index, reduction, scale)
    bad = int((valid & ((t < 0) | (t >= V))).sum())
    if bad:
        loss = np.full(N, np.nan) if reduction == NONE else float("nan")
        return dict(loss=loss, dX=None, dW=None, lse=None, n_valid=n_valid, bad_targets=bad)
    loss_rows = np.zeros(N)
    lse = np.zeros(N)
    dX = np.zeros((N, H)) if need_grads else None
    dW = np.zeros((V, H)) if need_grads else None
    for s in range(0, N, block_rows):
        e = min(N, s + block_rows)
        l_b, lse_b, dX_b, G_b = rows(X[s:e], W, t[s:e], coef[s:e], ignore_index)
        loss_rows[s:e] = l_b
        lse[s:e] = lse_b
        if need_grads:
            dX[s:e] = dX_b
            dW += G_b.T @ X[s:e]
    if reduction == SUM:
        loss = float(loss_rows.sum())
    elif reduction == MEAN:
        loss = float(loss_rows.sum() / n_valid) if n_valid > 0 else 0.0
    else:
        loss = loss_rows
    return dict(loss=loss, dX=dX, dW=dW, lse=lse, n_valid=n_valid, bad_targets=0)


def coef_for(t, ignore_index: int, reduction: str, scale: float):
    """Public helper: (valid mask, n_valid, coef) as defined in c3."""
    return _coef(np.asarray(t).astype(np.int64), ignore_index, reduction, scale)


def shard_stats(X, W_shard, t, vocab_start: int, ignore_index: int = -100):
    """Per-shard row statistics (m, s, z_t) of the vocab-sharded reading (R8).

    m_i = max over the shard's columns, s_i = sum exp(Z - m_i) over them, and
    z_t,i = Z_{i,t_i} if t_i falls in [vocab_start, vocab_start + V_l), else 0.
    Used only to pin the shard-combination identity.
    """
    X = np.asarray(X, dtype=np.float64)
    Z = X @ np.asarray(W_shard, dtype=np.float64).T
    m = Z.max(axis=1)
    s = np.exp(Z - m[:, None]).sum(axis=1)
    t = np.asarray(t).astype(np.int64)
    loc = t - vocab_start
    hit = (t != ignore_index) & (loc >= 0) & (loc < Z.shape[1])
    z_t = np.where(hit, Z[np.arange(Z.shape[0]), np.clip(loc, 0, Z.shape[1] - 1)], 0.0)
    return m, s, z_t


def combine_shards(stats):
    """lse and z_t from a list of shard (m, s, z_t): lse = M + log sum_k s_k e^{m_k - M}."""
    ms = np.stack([st[0] for st in stats])
    ss = np.stack([st[1] for st in stats])
    M = ms.max(axis=0)
    lse = M + np.log((ss * np.exp(ms - M)).sum(axis=0))
    z_t = np.stack([st[2] for st in stats]).sum(axis=0)
    return lse, z_t


def lce_output_memory(b: int, s: int, V: int, chunk_rows: int = 1024, elem_bytes: int = 2):
    """SPEC.md lines 146-154 memory model (logits + logit grads), for the report only."""
    full = b * s * V * elem_bytes * 2
    chunked = 2 * chunk_rows * V * elem_bytes
    return full, chunked, 1.0 - chunked / full


# ---- the final RMSNorm feeding the LM head (PAPER.md l.273 lists RMSNorm among
# the Triton kernels next to the fused LCE).  Plain definitions in float64.
def rmsnorm(x, g, eps: float = 1e-5):
    """y = x / sqrt(mean_h x^2 + eps) * g.  Returns (y, rstd)."""
    x = np.asarray(x, dtype=np.float64)
    rstd = 1.0 / np.sqrt((x * x).mean(axis=1) + eps)
    return x * rstd[:, None] * np.asarray(g, dtype=np.float64)[None, :], rstd


def rmsnorm_vjp(x, g, dy, eps: float = 1e-5):
    """Vector-Jacobian product of rmsnorm at x for the cotangent dy: (dx, dg).

    With xhat = x * rstd:  dx = rstd * (g*dy - xhat * mean_h(xhat * g * dy)),  dg = sum_rows dy * xhat.
    """
    x = np.asarray(x, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    dy = np.asarray(dy, dtype=np.float64)
    _, rstd = rmsnorm(x, g, eps)
    xhat = x * rstd[:, None]
    gdy = g[None, :] * dy
    c = (xhat * gdy).mean(axis=1)
    dx = rstd[:, None] * (gdy - xhat * c[:, None])
    dg = (dy * xhat).sum(axis=0)
    return dx, dg


def rmsnorm_lce(x, g, W, t, eps: float = 1e-5, **kw):
    """rmsnorm then lce: (loss, dx, dg, dW)."""
    y, _ = rmsnorm(x, g, eps)
    out = lce(y, W, t, **kw)
    dx, dg = rmsnorm_vjp(x, g, out["dX"], eps)
    return out["loss"], dx, dg, out["dW"]
