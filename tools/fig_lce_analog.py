"""B200 analog of the paper's Fig. fig:lce ("Memory usage and execution time
comparison between torch standard method and LCE for Llama3.1-8B") — context, not a target.

Times one forward+backward of the Llama-3.1-8B LM head + cross-entropy three ways on the same
synthetic inputs and reports time and peak extra device memory:
  * torch standard method: bf16 logits = X @ W^T, F.cross_entropy (fp32 upcast inside), autograd;
  * liger_kernel's Triton fused linear cross entropy (prior art, if importable);
  * this library (slf_lce_fwd_bwd, schedule AUTO).

    python tools/fig_lce_analog.py [--config llama8b] [--iters 5]
Writes one JSON line to stdout.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402


def measure(fn, iters):
    fn()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters, torch.cuda.max_memory_allocated() - base


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    N, H, V = c["N"], c["H"], c["V"]
    inp = synth.make_inputs(N, H, V, seed=0)
    X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda()
    t = torch.from_numpy(inp.t).cuda().long()
    out = {"config": a.config, "N": N, "H": H, "V": V, "logits_bytes": N * V * 2}

    Xg = X.clone().requires_grad_(True)
    Wg = W.clone().requires_grad_(True)

    def torch_std():
        Xg.grad = None
        Wg.grad = None
        loss = torch.nn.functional.cross_entropy((Xg @ Wg.T).float(), t, ignore_index=-100)
        loss.backward()

    try:
        ms, mem = measure(torch_std, a.iters)
        out["torch_standard"] = {"ms": ms, "peak_extra_bytes": mem}
    except torch.cuda.OutOfMemoryError as e:
        out["torch_standard"] = {"error": str(e)[:200]}
    torch.cuda.empty_cache()

    try:
        from liger_kernel.ops.fused_linear_cross_entropy import LigerFusedLinearCrossEntropyFunction as L

        def liger():
            Xg.grad = None
            Wg.grad = None
            loss = L.apply(Xg, Wg, t)
            loss = loss[0] if isinstance(loss, tuple) else loss
            loss.backward()

        ms, mem = measure(liger, a.iters)
        out["liger_flce_triton"] = {"ms": ms, "peak_extra_bytes": mem}
    except Exception as e:  # noqa: BLE001 — optional prior-art comparison
        out["liger_flce_triton"] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    torch.cuda.empty_cache()

    ws = slf.alloc_workspace(N, H, V, X.device)
    loss = torch.empty(1, dtype=torch.float32, device="cuda")
    dX = torch.empty_like(X)
    dW = torch.empty_like(W)

    def ours():
        slf.lce_fwd_bwd(X, W, t, out=(loss, dX, dW), workspace=ws)

    ms, mem = measure(ours, a.iters)
    out["slf_lce"] = {"ms": ms, "peak_extra_bytes": mem + ws.numel(), "workspace_bytes": ws.numel(),
                      "plan": slf.plan_describe(N, H, V)}
    flops = 6.0 * N * H * V
    for k in ("torch_standard", "liger_flce_triton", "slf_lce"):
        if "ms" in out.get(k, {}):
            out[k]["tflops_6NHV"] = flops / (out[k]["ms"] / 1e3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
