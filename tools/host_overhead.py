"""Host-side enqueue time of one fused call (no GPU sync inside the timed region); a rough check of
how much CPU work each step adds when the caller synchronises every step (bench e2e)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402


def main():
    c = synth.CONFIGS["llama8b"]
    N, H, V = c["N"], c["H"], c["V"]
    inp = synth.make_inputs(N, H, V, seed=0)
    X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda()
    t = torch.from_numpy(inp.t).cuda()
    ws = slf.alloc_workspace(N, H, V, X.device)
    loss = torch.empty(1, dtype=torch.float32, device="cuda")
    dX, dW = torch.empty_like(X), torch.empty_like(W)
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        slf.lce_fwd_bwd(X, W, t, out=(loss, dX, dW), workspace=ws)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"call {i}: enqueue {1e3 * (t1 - t0):.3f} ms, enqueue+run {1e3 * (t2 - t0):.3f} ms")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def per_step_sync_compare(steps=10):
    """Device call vs host-input call, both synchronised every step (events around the loop)."""
    c = synth.CONFIGS["llama8b"]
    N, H, V = c["N"], c["H"], c["V"]
    inp = synth.make_inputs(N, H, V, seed=0)
    X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda()
    t = torch.from_numpy(inp.t).cuda()
    Xh = X.cpu().pin_memory()
    th = t.cpu().pin_memory()
    lh = torch.empty(1, dtype=torch.float32).pin_memory()
    ws = slf.alloc_workspace(N, H, V, X.device)
    loss = torch.empty(1, dtype=torch.float32, device="cuda")
    dX, dW = torch.empty_like(X), torch.empty_like(W)
    stg = slf.HostStaging(N, H, X.device)
    s = torch.cuda.current_stream()

    def dev_step():
        slf.lce_fwd_bwd(X, W, t, out=(loss, dX, dW), workspace=ws)

    def host_step():
        slf.lce_fwd_bwd_host(Xh, W, th, dX=dX, dW=dW, loss_host=lh, staging=stg, workspace=ws)

    def torch_copy_step():
        stg.hidden.copy_(Xh, non_blocking=True)
        stg.targets.copy_(th, non_blocking=True)
        slf.lce_fwd_bwd(stg.hidden, W, stg.targets, out=(loss, dX, dW), workspace=ws)
        lh.copy_(loss, non_blocking=True)

    for name, fn, sync in (("device, no sync", dev_step, False), ("device, sync/step", dev_step, True),
                           ("host-input call, sync/step", host_step, True),
                           ("torch copies + device call, sync/step", torch_copy_step, True),
                           ("host-input call, no sync", host_step, False)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(steps):
            fn()
            if sync:
                s.synchronize()
        e1.record(s)
        torch.cuda.synchronize()
        print(f"{name:40s} {e0.elapsed_time(e1) / steps:.3f} ms/step")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--compare":
    per_step_sync_compare()
