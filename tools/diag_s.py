"""Diagnostic timing of the fused call's phases (not a bench line): which GEMM problem costs what.

    python tools/diag_s.py [--config llama8b] [--schedule S] [--budget-mult 1]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402
import paper_2603_16428_b200._lib as _L  # noqa: E402

if os.environ.get("SLF_SO"):  # experiment builds (tools/exp)
    _L.SO_PATH = os.environ["SLF_SO"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--schedule", default="S")
    ap.add_argument("--budget-mult", type=float, default=1.0)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    N, H, V = c["N"], c["H"], c["V"]
    inp = synth.make_inputs(N, H, V, seed=0)
    X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda()
    t = torch.from_numpy(inp.t).cuda()
    budget = int(max(0.05 * N * V * 2, 16 << 20) * a.budget_mult)
    print(slf.plan_describe(N, H, V, schedule=a.schedule, budget_bytes=budget))
    ws = slf.alloc_workspace(N, H, V, X.device, schedule=a.schedule, budget_bytes=budget)
    for name, ndx, ndw in (("full", True, True), ("dX only", True, False), ("dW only", False, True),
                           ("fwd only", False, False)):
        for _ in range(2):
            slf.lce_fwd_bwd(X, W, t, need_dhidden=ndx, need_dweight=ndw, workspace=ws, schedule=a.schedule,
                            budget_bytes=budget)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with slf.Profile() as p:
            e0.record()
            for _ in range(a.iters):
                slf.lce_fwd_bwd(X, W, t, need_dhidden=ndx, need_dweight=ndw, workspace=ws, schedule=a.schedule,
                                budget_bytes=budget)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        ks = ", ".join(f"{k} {v['ms'] / a.iters:.2f}ms" + (f" {v['flops'] / (v['ms'] / 1e3) / 1e12:.0f}TF" if v['flops'] else "")
                       for k, v in p.kinds.items())
        print(f"{name:9s} {ms:7.2f} ms | {ks}", flush=True)


if __name__ == "__main__":
    main()
