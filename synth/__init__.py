"""Seeded synthetic inputs for the fused linear-cross-entropy (LCE) hot path.

This module is shared by the oracle side (tests, ``oracle/``) and the CUDA side
(tests, ``bench.py``).  It holds NO arithmetic of the method: it only draws
random numbers and rounds them to bf16 bit patterns.  Recipe (DESIGN.md §Inputs,
SURVEY.md §8(d) row d2):

* ``X`` ~ N(0, 1) rounded to bf16 (unit-RMS hidden states, like the output of a
  final RMSNorm).
* ``W`` ~ N(0, alpha^2 / H) rounded to bf16, so logits have std ~= alpha.
  alpha = 1 is init-like (flat softmax, loss ~= ln V), alpha = 4 trained-like
  (peaked softmax).
* ``targets`` uniform on [0, V) or Zipf(s=1.1) by rank (rank -> id through a
  seeded permutation, so hot vocabulary rows are scattered over the shard).
* ignore: exactly round(ignore_frac * N) positions chosen by a seeded
  permutation are set to ``ignore_index`` (default -100).

Seeds: ``seed`` is the base; X, W, targets and ignore positions use
``seed + 1``, ``seed + 2``, ``seed + 3``, ``seed + 4`` of numpy's PCG64.

bf16 values are returned as ``uint16`` bit patterns (numpy has no bf16 type);
``bf16_bits_to_f64`` turns them into exact float64 values.
"""
from __future__ import annotations

import dataclasses

import numpy as np

# BASELINE.json "configs" (N tokens, H hidden, V vocab).
CONFIGS = {
    "tiny": dict(N=256, H=512, V=4096),
    "llama8b": dict(N=16384, H=4096, V=128256),
    "qwen7b": dict(N=32768, H=3584, V=152064),
    "llama70b": dict(N=65536, H=8192, V=128256),
    "mistral123b": dict(N=65536, H=12288, V=32768),
}


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); return the bits.

    Inputs here are finite normal draws, so no NaN handling is needed.
    """
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rounding = np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    return ((u + rounding) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    """Exact: every bf16 value is representable in float64."""
    return bf16_bits_to_f32(b).astype(np.float64)


def _normal_bf16(rng: np.random.Generator, shape, std: float, chunk: int = 1 << 26) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.uint16)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        v = rng.standard_normal(e - s, dtype=np.float32)
        if std != 1.0:
            v *= np.float32(std)
        out[s:e] = f32_to_bf16_bits(v)
    return out.reshape(shape)


def zipf_targets(rng: np.random.Generator, n: int, V: int, s: float = 1.1) -> np.ndarray:
    ranks = np.arange(1, V + 1, dtype=np.float64)
    p = ranks ** (-s)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    r = np.searchsorted(cdf, rng.random(n), side="right")
    r = np.minimum(r, V - 1)
    perm = rng.permutation(V)
    return perm[r].astype(np.int32)


@dataclasses.dataclass
class LCEInputs:
    X: np.ndarray  # [N, H] uint16 (bf16 bits)
    W: np.ndarray  # [V, H] uint16 (bf16 bits)
    t: np.ndarray  # [N] int32
    ignore_index: int
    N: int
    H: int
    V: int


def make_targets(N: int, V: int, seed: int = 0, dist: str = "uniform", ignore_frac: float = 0.05,
                 ignore_index: int = -100) -> np.ndarray:
    rng_t = np.random.Generator(np.random.PCG64(seed + 3))
    if dist == "uniform":
        t = rng_t.integers(0, V, size=N, dtype=np.int64).astype(np.int32)
    elif dist == "zipf":
        t = zipf_targets(rng_t, N, V)
    else:
        raise ValueError(f"unknown target distribution {dist!r}")
    n_ign = int(round(ignore_frac * N))
    if n_ign:
        rng_i = np.random.Generator(np.random.PCG64(seed + 4))
        pos = rng_i.permutation(N)[:n_ign]
        t[pos] = ignore_index
    return t


def make_inputs(N: int, H: int, V: int, seed: int = 0, alpha: float = 1.0, dist: str = "uniform",
                ignore_frac: float = 0.05, ignore_index: int = -100, with_w: bool = True) -> LCEInputs:
    rng_x = np.random.Generator(np.random.PCG64(seed + 1))
    rng_w = np.random.Generator(np.random.PCG64(seed + 2))
    X = _normal_bf16(rng_x, (N, H), 1.0)
    W = _normal_bf16(rng_w, (V, H), alpha / np.sqrt(H)) if with_w else None
    t = make_targets(N, V, seed, dist, ignore_frac, ignore_index)
    return LCEInputs(X=X, W=W, t=t, ignore_index=ignore_index, N=N, H=H, V=V)


def make_config(name: str, seed: int = 0, alpha: float = 1.0, dist: str = "uniform", N: int | None = None,
                ignore_frac: float = 0.05) -> LCEInputs:
    c = dict(CONFIGS[name])
    if N is not None:
        c["N"] = N
    return make_inputs(c["N"], c["H"], c["V"], seed=seed, alpha=alpha, dist=dist, ignore_frac=ignore_frac)
