"""Fused final RMSNorm + LCE (slf_rmsnorm_lce_fwd_bwd) against the composition rmsnorm_fwd ->
lce_fwd_bwd -> rmsnorm_bwd at an LM-head shape.

    python tools/bench_rmsnorm_lce.py [--config llama8b] [--steps 10] [--pairs 5]

Both arms use preallocated outputs and workspaces (the composition also its y [N, H] buffer, rstd
and the RMSNorm backward workspace), W warm-ups, then `pairs` alternating timed blocks of `steps`
steps each (CUDA events on the current stream).  Prints one JSON line.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402
from paper_2603_16428_b200 import lce as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b", choices=list(synth.CONFIGS))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--pairs", type=int, default=5)
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    N, H, V = c["N"], c["H"], c["V"]
    inp = synth.make_inputs(N, H, V, seed=0, alpha=1.0)
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).to(dev)
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).to(dev)
    t = torch.from_numpy(inp.t).to(dev)
    g = (1 + 0.1 * torch.randn(H, generator=torch.Generator().manual_seed(0))).to(torch.bfloat16).to(dev)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    dx = torch.empty_like(x)
    dg = torch.empty(H, dtype=torch.float32, device=dev)
    dW = torch.empty_like(W)
    ws_f = torch.empty(slf.rmsnorm_lce_workspace_bytes(N, H, V), dtype=torch.uint8, device=dev)
    ws_l = slf.alloc_workspace(N, H, V, dev)
    y = torch.empty_like(x)
    rstd = torch.empty(N, dtype=torch.float32, device=dev)
    ws_r = torch.empty(slf.rmsnorm_workspace_bytes(N, H), dtype=torch.uint8, device=dev)
    s = L._stream_ptr(dev)

    def fused():
        slf.rmsnorm_lce_fwd_bwd(x, g, W, t, out=(loss, dx, dg, dW), workspace=ws_f)

    def composed():
        L.check(L.lib().slf_rmsnorm_fwd(x.data_ptr(), g.data_ptr(), N, H, 1e-5, y.data_ptr(), rstd.data_ptr(), s),
                "slf_rmsnorm_fwd")
        slf.lce_fwd_bwd(y, W, t, out=(loss, dx, dW), workspace=ws_l)
        slf.rmsnorm_bwd(x, g, rstd, dx, dx=dx, workspace=ws_r, dg=dg)

    res = {"fused": [], "composed": []}
    for f in (fused, composed):
        for _ in range(a.warmup):
            f()
    torch.cuda.synchronize()
    for _ in range(a.pairs):
        for name, f in (("fused", fused), ("composed", composed)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                f()
            e1.record()
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) / a.steps)
    with slf.Profile() as pf:
        for _ in range(a.steps):
            fused()
        torch.cuda.synchronize()
    rms_f = {k: v["ms"] / a.steps for k, v in pf.kinds.items()}
    with slf.Profile() as pc:
        for _ in range(a.steps):
            composed()
        torch.cuda.synchronize()
    rms_c = {k: v["ms"] / a.steps for k, v in pc.kinds.items()}
    out = {
        "workload": f"{a.config} final RMSNorm + LM head N={N} H={H} V={V}",
        "fused_ms": res["fused"], "composed_ms": res["composed"],
        "fused_ms_median": float(np.median(res["fused"])), "composed_ms_median": float(np.median(res["composed"])),
        "saved_ms_median": float(np.median(np.array(res["composed"]) - np.array(res["fused"]))),
        "nh_roundtrip_ms_at_hbm_peak": N * H * 2 * 4 / 6.5e12 * 1e3,
        "kernel_ms_per_step": {"fused": rms_f, "composed": rms_c},
        "extra_device_bytes": {"fused_workspace": ws_f.numel(),
                               "composed": ws_l.numel() + y.numel() * 2 + rstd.numel() * 4 + ws_r.numel()},
        "plan": slf.rmsnorm_lce_plan_describe(N, H, V),
        "note": "alternating blocks of steps; saved_ms = per-pair composed - fused; the N*H round trip is the y "
                "write + read and the dy read + write the fused call avoids (4 * N*H*2 bytes at 6.5 TB/s)",
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
