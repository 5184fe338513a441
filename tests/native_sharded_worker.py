"""One rank of the native vocab-sharded call (slf_lce_fwd_bwd_sharded) with a callback transport:
gloo collectives through host copies, so g ranks can share ONE GPU (NCCL refuses two ranks on one
device).  Launched g times by tests/test_gpu_parity.py::test_native_sharded_callbacks; writes this
rank's loss, dhidden and dW rows to <out>/rank<r>.npz.  The library's orchestration (chunk loop,
double-buffered dX partials, all-gather / all-reduce order) is what runs; only the byte transport
is the test's.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_2603_16428_b200 as slf  # noqa: E402


class _Raw:
    """A device byte range as a torch tensor (__cuda_array_interface__)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": typestr,
                                         "version": 3, "strides": None}


def raw(ptr, n, typestr="|u1"):
    return torch.as_tensor(_Raw(ptr, n, typestr), device="cuda")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--N", type=int, default=900)
    ap.add_argument("--H", type=int, default=256)
    ap.add_argument("--V", type=int, default=5000)
    ap.add_argument("--budget", type=int, default=3 << 20)
    ap.add_argument("--reduction", default="mean")
    ap.add_argument("--ignore-index", type=int, default=-100)
    ap.add_argument("--p2p", type=int, default=0, help="P2P exchanges over IPC: 1 statistics, 2 dX, 3 both")
    ap.add_argument("--calls", type=int, default=1, help="calls on the same communicator (the last is saved)")
    ap.add_argument("--mode", default="vocab", choices=["vocab", "dp"],
                    help="vocab: slf_lce_fwd_bwd_sharded; dp: slf_lce_fwd_bwd_dp on this rank's tokens")
    a = ap.parse_args()
    dist.init_process_group("gloo", rank=a.rank, world_size=a.world)
    torch.cuda.set_device(0)
    calls = {"ag": 0, "ar": 0}

    def allgather(send, recv, nbytes, stream):
        torch.cuda.synchronize()
        s = raw(send, nbytes).cpu()
        parts = [torch.empty_like(s) for _ in range(a.world)]
        dist.all_gather(parts, s)
        raw(recv, nbytes * a.world).copy_(torch.cat(parts).cuda())
        torch.cuda.synchronize()
        calls["ag"] += 1

    def allreduce(buf, count, stream):
        torch.cuda.synchronize()
        b = raw(buf, count, "<f4").cpu()
        dist.all_reduce(b)
        raw(buf, count, "<f4").copy_(b.cuda())
        torch.cuda.synchronize()
        calls["ar"] += 1

    inp = synth.make_inputs(a.N, a.H, a.V, seed=21, alpha=4.0, dist="zipf", ignore_index=a.ignore_index)
    X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda()
    t = torch.from_numpy(inp.t.astype(np.int32)).cuda()
    v0, v1 = slf.shard_bounds_native(a.V, a.world, a.rank)
    comm = slf.Comm.callbacks(a.rank, a.world, allgather, allreduce)
    if a.p2p:
        comm.set_p2p(a.p2p)
    Wl = W[v0:v1].contiguous()
    n0, n1 = a.N * a.rank // a.world, a.N * (a.rank + 1) // a.world
    for _ in range(a.calls):
        calls["ag"] = calls["ar"] = 0
        if a.mode == "dp":
            loss, dX, dW = slf.lce_fwd_bwd_dp(X[n0:n1].clone(), W, t[n0:n1].clone(), comm,
                                              ignore_index=a.ignore_index, reduction=a.reduction,
                                              budget_bytes=a.budget)
            v0, v1 = n0, n1  # saved: this rank's token rows
        else:
            loss, dX, dW = slf.lce_fwd_bwd_sharded(X, Wl, t, a.V, comm, ignore_index=a.ignore_index,
                                                   reduction=a.reduction, budget_bytes=a.budget)
        torch.cuda.synchronize()
    timeouts = comm.p2p_timeouts()
    comm.close()
    np.savez(os.path.join(a.out, f"rank{a.rank}.npz"), loss=loss.detach().cpu().numpy(),
             dX=dX.view(torch.int16).cpu().numpy(), dW=dW.view(torch.int16).cpu().numpy(), v0=v0, v1=v1,
             ag=calls["ag"], ar=calls["ar"], timeouts=timeouts,
             plan=slf.sharded_plan_describe(a.N, a.H, a.V, a.world, a.rank, a.budget) if a.mode == "vocab" else "dp")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
