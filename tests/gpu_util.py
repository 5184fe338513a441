"""Helpers shared by the GPU parity tests: move synth inputs to the device, compare with the oracle."""
import numpy as np

import synth


def to_dev(inp, torch):
    X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda() if inp.W is not None else None
    t = torch.from_numpy(inp.t.astype(np.int32)).cuda()
    return X, W, t


def bf16_to_np64(t):
    import torch
    return t.detach().float().cpu().numpy().astype(np.float64) if t.dtype == torch.bfloat16 else \
        t.detach().cpu().numpy().astype(np.float64)


def rel_max_err(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    got = np.asarray(got, dtype=np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(got - ref)) / (den if den > 0 else 1.0))


# Tolerances from BASELINE.json north_star: loss relative 1e-3; dX, dW max|err| <= 2e-2 max|ref|.
LOSS_RTOL = 1e-3
GRAD_TOL = 2e-2


def assert_loss_close(got, ref, reduction):
    if reduction == "none":
        got = np.asarray(got, dtype=np.float64)
        ref = np.asarray(ref, dtype=np.float64)
        floor = 1e-3 * max(np.max(np.abs(ref)), 1e-30)
        err = np.abs(got - ref)
        bad = err > np.maximum(LOSS_RTOL * np.abs(ref), floor)
        assert not bad.any(), f"per-row loss mismatch at {np.nonzero(bad)[0][:10]} max err {err.max()}"
    else:
        assert abs(float(got) - float(ref)) <= LOSS_RTOL * abs(float(ref)) + 1e-30, (float(got), float(ref))


def oracle_inputs(inp):
    return synth.bf16_bits_to_f64(inp.X), synth.bf16_bits_to_f64(inp.W), inp.t.astype(np.int64)
