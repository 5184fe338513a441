"""Where the end-to-end (host-input) step loses time against the device-resident step: the same
loop with (a) the device call, (b) the device call + a separate pinned H2D of hidden/targets on a
side stream, (c) the host-input call with one staging set, (d) with two staging sets."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402

c = synth.CONFIGS["llama8b"]
N, H, V = c["N"], c["H"], c["V"]
inp = synth.make_inputs(N, H, V, seed=0)
dev = torch.device("cuda", 0)
X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).to(dev)
W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).to(dev)
t = torch.from_numpy(inp.t).to(dev)
Xh = X.cpu().pin_memory()
th = t.cpu().pin_memory()
ws = slf.alloc_workspace(N, H, V, dev)
loss = torch.empty(1, device=dev)
dX = torch.empty_like(X)
dW = torch.empty_like(W)
lh = [torch.empty(1).pin_memory() for _ in range(2)]
stg = [slf.HostStaging(N, H, dev) for _ in range(2)]
side = torch.cuda.Stream()


def run(mode, steps=10):
    done = [torch.cuda.Event() for _ in range(2)]
    cur = torch.cuda.current_stream()

    def one(i):
        k = i % 2
        if mode == "device":
            slf.lce_fwd_bwd(X, W, t, out=(loss, dX, dW), workspace=ws)
            lh[k].copy_(loss, non_blocking=True)
        elif mode == "device+copy":
            with torch.cuda.stream(side):
                stg[k].hidden.copy_(Xh, non_blocking=True)
                stg[k].targets.copy_(th, non_blocking=True)
            slf.lce_fwd_bwd(X, W, t, out=(loss, dX, dW), workspace=ws)
            lh[k].copy_(loss, non_blocking=True)
        else:
            s = stg[k] if mode == "host2" else stg[0]
            slf.lce_fwd_bwd_host(Xh, W, th, dX=dX, dW=dW, loss_host=lh[k], staging=s, workspace=ws)
        done[k].record(cur)
        if i > 0:
            done[1 - k].synchronize()

    for i in range(3):
        one(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(steps):
        one(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, (time.perf_counter() - t0) * 1e3 / steps


for rep in range(2):
    for mode in ("device", "device+copy", "host1", "host2"):
        ev, wall = run(mode)
        print(f"{mode:12s} events {ev:.2f} ms  wall {wall:.2f} ms")
