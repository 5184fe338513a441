"""Timed fine-tuning steps of the LM-head block at an LM-head shape:
LMHeadTrainer.step = fused RMSNorm + LCE on the GPU, then Layer-Adam on the host for W (device-fed).

    python tools/bench_train_step.py [--config llama8b] [--steps 6] [--warmup 2]

Fresh synthetic batches (N tokens each) are staged on the device before timing.  Reports wall time
per step (host perf_counter around K steps ending in finish(); the host Adam update is on the
critical path), the GPU part alone (CUDA events around the fused call, same loop), tokens/s, and
the loss trajectory.  One JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402
from paper_2603_16428_b200.train import LMHeadTrainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b", choices=list(synth.CONFIGS))
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--lr", type=float, default=1e-4)
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    N, H, V = c["N"], c["H"], c["V"]
    dev = torch.device("cuda", 0)
    base = synth.make_inputs(N, H, V, seed=0, alpha=4.0, dist="zipf")
    W = torch.from_numpy(base.W.view(np.int16)).view(torch.bfloat16).to(dev)
    g = (1 + 0.1 * torch.randn(H, generator=torch.Generator().manual_seed(0))).to(torch.bfloat16).to(dev)
    nb = 2
    batches = []
    for k in range(nb):
        b = synth.make_inputs(N, H, V, seed=100 + k, alpha=4.0, dist="zipf", with_w=False)
        batches.append((torch.from_numpy(b.X.view(np.int16)).view(torch.bfloat16).to(dev),
                        torch.from_numpy(b.t).to(dev)))
    t0 = time.perf_counter()
    tr = LMHeadTrainer(W, g, lr=a.lr)
    init_s = time.perf_counter() - t0
    for k in range(a.warmup):
        tr.step(*batches[k % nb])
    tr.finish()
    torch.cuda.synchronize()
    losses, gpu_ms = [], []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    w0 = time.perf_counter()
    for k in range(a.steps):
        loss, dx, dg = tr.step(*batches[k % nb], events=ev[k])
        losses.append(loss.clone())
    tr.finish()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) / a.steps
    gpu_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    out = {
        "workload": f"{a.config} LM-head training step N={N} H={H} V={V}: fused RMSNorm+LCE (GPU) + Layer-Adam on W "
                    f"(host, device-fed)",
        "ms_per_step_wall": wall * 1e3, "tokens_per_s": N / wall,
        "gpu_fused_ms_median": float(np.median(gpu_ms)),
        "host_adam_share": 1.0 - float(np.median(gpu_ms)) / (wall * 1e3),
        "losses": [float(x) for x in losses], "steps": a.steps, "warmup": a.warmup,
        "adam_init_s": init_s, "cpu_threads": torch.get_num_threads(), "simd_width": slf.adam.simd_width(),
        "note": "wall time per step over K steps (the host Adam update of step k overlaps nothing: step k+1 reads "
                "the updated W); GPU time = CUDA events around each fused call",
    }
    print(json.dumps(out))
    tr.close()


if __name__ == "__main__":
    main()
