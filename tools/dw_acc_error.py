"""dW / dX error against the fp64 oracle for the dW accumulation modes (SLF_DW_ACC=2, default: L2 reduce-add of a bf16 partial; 1: load-add-store
in the epilogue, one rounding).  Run once per mode.

    SLF_DW_ACC=2 python tools/dw_acc_error.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402
from gpu_util import bf16_to_np64, oracle_inputs, rel_max_err, to_dev  # noqa: E402


def main():
    for (N, H, V, budget, dist, alpha) in ((4096, 1024, 16384, 10 << 20, "zipf", 4.0),
                                           (4096, 1024, 16384, 10 << 20, "uniform", 1.0),
                                           (8192, 512, 8192, 5 << 20, "zipf", 4.0)):
        inp = synth.make_inputs(N, H, V, seed=7, alpha=alpha, dist=dist)
        X, W, t = to_dev(inp, torch)
        desc = slf.plan_describe(N, H, V, schedule="S", budget_bytes=budget)
        loss, dX, dW = slf.lce_fwd_bwd(X, W, t, reduction="mean", schedule="S", budget_bytes=budget)
        torch.cuda.synchronize()
        Xo, Wo, to = oracle_inputs(inp)
        ref = oracle.lce(Xo, Wo, to, reduction="mean")
        print(f"mode {os.environ.get('SLF_DW_ACC', '2')} N={N} H={H} V={V} {dist} a={alpha} [{desc}]: "
              f"dX {rel_max_err(bf16_to_np64(dX), ref['dX']):.2e} dW {rel_max_err(bf16_to_np64(dW), ref['dW']):.2e}")


if __name__ == "__main__":
    main()
