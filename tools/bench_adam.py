"""Layer-Adam measurement at an LM-head size: host-step throughput against
the host's memory bandwidth (STREAM-style copy / add over all host threads, same run), and the
device-fed pipelined step (d2h of dW, CPU update, h2d of the bf16 W) against its three stages run back to back.  Prints one JSON line.

    python tools/bench_adam.py --config llama8b --steps 3

Algorithmic bytes per element of a host step: read bf16 g (2) + fp32 p, m, v (12), write p, m, v
(12) + bf16 param copy (2) = 28 B.  The bandwidth denominator is a STREAM-style copy / add split
over all host threads on buffers far larger than the caches, measured in the same run.
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2603_16428_b200.adam import LayerAdam, simd_width  # noqa: E402


def host_stream_gbs(nbytes: int, reps: int = 3) -> dict:
    """STREAM-style host bandwidth: copy (c = a) and add (c = a + b), each split over all host threads
    (numpy releases the GIL on large slices).  DRAM bytes per second counting the write-allocate
    read of c (plain stores, as in the Adam update, whose p, m, v stores hit lines it has just read):
    copy moves 3 x nbytes, add 4 x nbytes."""
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np
    nt = len(os.sched_getaffinity(0))
    n = nbytes // 4
    a = np.ones(n, dtype=np.float32)
    b = np.ones(n, dtype=np.float32)
    c = np.zeros(n, dtype=np.float32)
    cuts = [n * k // nt for k in range(nt + 1)]
    sl = [slice(cuts[k], cuts[k + 1]) for k in range(nt)]
    res = {}
    with ThreadPoolExecutor(nt) as ex:
        for name, fn, rw in (("copy", lambda s: np.copyto(c[s], a[s]), 3),
                             ("add", lambda s: np.add(a[s], b[s], out=c[s]), 4)):
            best = 0.0
            for _ in range(reps + 1):
                t0 = time.perf_counter()
                list(ex.map(fn, sl))
                best = max(best, rw * nbytes / (time.perf_counter() - t0) / 1e9)
            res[name] = best
    res["threads"] = nt
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b", choices=list(synth.CONFIGS))
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    n = c["V"] * c["H"]
    dev = torch.device("cuda", 0)
    opt = LayerAdam(n, lr=1e-4, weight_decay=0.01, threads=a.threads)
    W = (torch.randn(c["V"], c["H"], device=dev) * 0.02).bfloat16()
    opt.set_params(W.cpu())
    gh = (torch.randn(n) * 1e-3).bfloat16()
    out = torch.empty(n, dtype=torch.bfloat16)
    opt.step_host(gh, 1.0, out)  # warm-up (first touch)
    ts = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        opt.step_host(gh, 1.0, out)
        ts.append(time.perf_counter() - t0)
    t_host = min(ts)
    bw = host_stream_gbs(min(4 << 30, n * 8))

    # device-fed pipelined step
    gd = gh.to(dev)
    opt.step_device_async(gd, W.view(-1))
    opt.wait()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        opt.step_device_async(gd, W.view(-1))
        opt.wait()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t_dev = min(ts)
    # the stages one after the other (pinned copies with torch, the same host update)
    gp = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    op = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gp.copy_(gd)
    torch.cuda.synchronize()
    t_d2h = time.perf_counter() - t0
    t0 = time.perf_counter()
    opt.step_host(gp, 1.0, op)
    t_upd = time.perf_counter() - t0
    t0 = time.perf_counter()
    W.view(-1).copy_(op, non_blocking=True)
    torch.cuda.synchronize()
    t_h2d = time.perf_counter() - t0
    gbs = 28.0 * n / t_host / 1e9
    print(json.dumps({
        "component": "Layer-Adam (host, SURVEY §8(f) NEXT-4)", "config": a.config, "elements": n,
        "simd_width": simd_width(), "threads": a.threads or torch.get_num_threads(),
        "host_step_ms": t_host * 1e3, "host_step_gbs": gbs, "host_stream_gbs": bw,
        "frac_of_host_stream": gbs / max(bw["copy"], bw["add"]),
        "algorithmic_bytes_per_elem": 28,
        "device_fed_step_ms": t_dev * 1e3,
        "stages_serial_ms": {"d2h": t_d2h * 1e3, "update": t_upd * 1e3, "h2d": t_h2d * 1e3,
                             "sum": (t_d2h + t_upd + t_h2d) * 1e3},
        "overlap_gain": (t_d2h + t_upd + t_h2d) / t_dev,
        "pcie_gbs": {"d2h": 2 * n / t_d2h / 1e9, "h2d": 2 * n / t_h2d / 1e9},
    }), flush=True)
    opt.close()


if __name__ == "__main__":
    main()
