"""Benchmark of the fused linear-cross-entropy hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b] [--impl slf|reference]

One step = one full fused LCE forward + backward (loss, dL/dhidden, dL/dW_lmhead) over one batch of
synthetic inputs of the named LM-head shape (default: Llama-3.1-8B, N=16384 tokens, H=4096,
V=128256).  N=1: the single-GPU C-ABI call slf_lce_fwd_bwd.  N>1 (torchrun, one rank per GPU):
the vocab-sharded path (each rank owns V/N rows of W; NCCL all-gather of per-token statistics,
NCCL all-reduce of the fp32 dhidden partials; dW stays local) — strong scaling of the same call.

Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 CPU oracle (the reference arm of
this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "fused LCE fwd+bwd tokens/s and % BF16 tensor peak at 1/2/4/8 B200"
UNIT = "tokens/s"
L2_BYTES = 126 * 1024 * 1024


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return dict(burst=float(d["bf16_tflops"]), sustained=float(d["bf16_tflops_sustained"]),
                    hbm=float(d["hbm_gbs"]), source="MEASURED_PEAKS.json (measured)",
                    sustained_mhz=(d.get("clocks_under_load") or {}).get("sm_mhz_median"))
    except Exception:
        return dict(burst=1590.0, sustained=1400.0, hbm=6650.0, source="B200_PROFILING.md fallback",
                    sustained_mhz=None)


# ---- clocks sampler ---------------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self, t0=None, t1=None):
        """Samples taken inside [t0, t1] (perf_counter seconds; the timed region), else all."""
        sm, pw, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for ts, ln in self.lines if (t0 is None or ts >= t0) and (t1 is None or ts <= t1)]
        for ln in (inside or [ln for _, ln in self.lines]):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": float(np.median(pw)) if pw else None,
                "power_w_max": float(np.max(pw)) if pw else None}


# ---- oracle timing (cpu_baseline and --impl reference) ---------------------------------------------
def oracle_sample_time(inp_X, W64, t, rows: int):
    import oracle
    Xs = synth.bf16_bits_to_f64(inp_X[:rows])
    ts = t[:rows].astype(np.int64)
    t0 = time.perf_counter()
    oracle.lce(Xs, W64, ts, reduction="sum", scale=1.0 / max(1, rows), block_rows=rows)
    return time.perf_counter() - t0


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        th = max((d.get("num_threads", 1) for d in threadpool_info() if d.get("user_api") == "blas"), default=1)
    except Exception:
        th = None
    return th or len(os.sched_getaffinity(0))


def oracle_rows_for(inp_X, W64, t, seconds: float, cap: int) -> int:
    """Rows of a bounded oracle sample taking about `seconds`: the oracle has a fixed per-call cost
    (its fp64 [V, H] dW), so fit time = a + b * rows from two sample sizes."""
    t8 = oracle_sample_time(inp_X, W64, t, 8)
    t32 = oracle_sample_time(inp_X, W64, t, 32)
    b = max((t32 - t8) / 24, 1e-6)
    a = max(t8 - 8 * b, 0.0)
    return int(np.clip((seconds - a) / b, 8, cap))


def cpu_info():
    """CPU model (lscpu / /proc/cpuinfo) and the BLAS numpy runs on (threadpoolctl): SURVEY §8(d) d7."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        b = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        if b:
            blas = f"{b[0].get('internal_api')} {b[0].get('version')} ({b[0].get('num_threads')} threads)"
    except Exception:
        pass
    return {"cpu_model": model, "blas": blas}


def cpu_baseline(inp, cfg_name, target_s=12.0):
    W64 = synth.bf16_bits_to_f64(inp.W)
    rows = oracle_rows_for(inp.X, W64, inp.t, target_s, min(2048, inp.N))
    dt = oracle_sample_time(inp.X, W64, inp.t, rows)
    return {"value": rows / dt, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
            "sample": f"{rows} tokens of the {cfg_name} workload at full H={inp.H}, V={inp.V} (numpy fp64, "
                      f"materialised logits; per-token work is 6*H*V so tokens/s extrapolates linearly)",
            "seconds": dt, **cpu_info()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    c = synth.CONFIGS[args.config]
    inp = synth.make_inputs(min(c["N"], 2048), c["H"], c["V"], seed=args.seed, alpha=args.alpha, dist=args.dist)
    W64 = synth.bf16_bits_to_f64(inp.W)
    rows = oracle_rows_for(inp.X, W64, inp.t, 3.0, inp.N)  # ~3 s of CPU work per step
    for _ in range(args.warmup):
        oracle_sample_time(inp.X, W64, inp.t, rows)
    times = [oracle_sample_time(inp.X, W64, inp.t, rows) for _ in range(args.steps)]
    dt = float(np.mean(times))
    v = rows / dt
    cores = cpu_cores()
    sample = f"{rows} tokens per step of the {args.config} workload (full H, V), numpy fp64 oracle"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} LM head N={c['N']} H={c['H']} V={c['V']} (oracle: bounded row sample)",
                   "N": c["N"], "H": c["H"], "V": c["V"], "sample_tokens": rows},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample, **cpu_info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---- the GPU arm -----------------------------------------------------------------------------------
def launcher_cmd(gpus: int, argv, port: int):
    """The command that runs this script with one rank per GPU (torch.distributed.run, loopback
    rendezvous), forwarding the original arguments."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(gpus: int) -> int:
    """Spawn `gpus` ranks of this benchmark; rank 0's JSON line reaches our stdout unchanged.  Fails
    loudly (exit 2) when fewer GPUs are visible than requested."""
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < gpus and "--dry-run" not in sys.argv[1:]:
        print(f"bench.py: --gpus {gpus} requested but {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    cmd = launcher_cmd(gpus, sys.argv[1:], free_port())
    print("bench.py: launching " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def run_dry(args):
    """The multi-rank plumbing of the GPU arm without a GPU: process group, barrier, max over ranks,
    rank 0 alone prints.  No measurement."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dist.barrier()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_over_ranks": float(t.item()),
                          "local_rank": int(os.environ.get("LOCAL_RANK", "0"))}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="slf", choices=["slf", "reference"])
    ap.add_argument("--config", default="llama8b", choices=list(synth.CONFIGS))
    ap.add_argument("--dist", default="uniform", choices=["uniform", "zipf"])
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--budget", type=int, default=0, help="workspace budget bytes (0 = 5%% of N*V*2)")
    ap.add_argument("--schedule", default="auto", choices=["auto", "R", "S"])
    ap.add_argument("--emulate-shards", type=int, default=0,
                    help="with --module at world size 1: time rank 0's vocab shard of G GPUs (no exchange)")
    ap.add_argument("--module", action="store_true",
                    help="run the multi-GPU module path (NCCL process group) even at world size 1 (testing)")
    ap.add_argument("--parallel", default="vocab", choices=["vocab", "dp"],
                    help="N>1: vocab-sharded W (north star) or token-sharded data parallel (full W per GPU)")
    ap.add_argument("--comm", default="native", choices=["native", "torch"],
                    help="vocab-sharded schedule S: collectives inside the library (slf_comm over NCCL, "
                         "slf_lce_fwd_bwd_sharded) or orchestrated from Python over torch.distributed")
    ap.add_argument("--comm-sms", type=int, default=-1,
                    help="native comm at N>1: SMs the GEMM launches leave to the communicator's kernels "
                         "(-1: the library default, 8)")
    ap.add_argument("--p2p-stats", action="store_true",
                    help="native comm: per-chunk statistics by the P2P one-shot all-gather over CUDA IPC (NEXT-3)")
    ap.add_argument("--p2p-dx", action="store_true",
                    help="native comm: dX exchanged by the P2P reduce/all-gather kernel over CUDA IPC (no NCCL)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher plumbing only (CPU tests): ranks join a gloo group, exchange a per-rank "
                         "number with the max-over-ranks reduction the timing uses, rank 0 prints it")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return

    # N > 1 without a launcher: start one rank per GPU ourselves (the same torch.distributed.run
    # command the driver uses), so `python bench.py --gpus N` is never silently a 1-GPU run.
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        sys.exit(self_launch(args.gpus))
    if world_env is not None and int(world_env) != args.gpus and not (args.gpus == 1 and args.module):
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}; refusing to time a different "
              f"configuration", file=sys.stderr)
        sys.exit(2)
    if args.dry_run:
        run_dry(args)
        return
    if args.gpus > 1 or world_env is not None:
        # NCCL's INIT lines (ranks, devices, channels, NVLS) on stderr: evidence of the ranks used
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

    if args.comm_sms >= 0:
        os.environ["SLF_COMM_SMS"] = str(args.comm_sms)
    # The JSON line is the only thing this process writes to stdout: libraries that print to the C
    # stdout (e.g. NCCL's version banner) are sent to stderr for the rest of the run.
    json_out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)

    import torch
    import torch.distributed as dist

    import paper_2603_16428_b200 as slf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    multi = world > 1 or args.module  # the multi-GPU code path (also at world size 1 with --module)
    if multi:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29547")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    g = world

    c = synth.CONFIGS[args.config]
    N, H, V = c["N"], c["H"], c["V"]
    inp = synth.make_inputs(N, H, V, seed=args.seed, alpha=args.alpha, dist=args.dist)
    dp = multi and args.parallel == "dp"
    G = args.emulate_shards if (args.emulate_shards and world == 1 and args.module and not dp) else g
    v0, v1 = (0, V) if dp else (V * rank // G, V * (rank + 1) // G)
    n0, n1 = (N * rank // g, N * (rank + 1) // g) if dp else (0, N)
    V_l = v1 - v0
    N_l = n1 - n0
    X = torch.from_numpy(inp.X[n0:n1].view(np.int16)).view(torch.bfloat16).to(dev)
    W = torch.from_numpy(inp.W[v0:v1].view(np.int16)).view(torch.bfloat16).to(dev)
    t = torch.from_numpy(inp.t[n0:n1]).to(dev)

    if multi and args.budget == 0 and not dp:
        # Sharded runs: 5% of the GLOBAL N*V*2 logits per GPU (SURVEY q7 "lenient" reading; both
        # ratios are reported in "memory").
        args.budget = int(0.05 * N * V * 2)
    ws_budget = args.budget
    if multi and not dp:
        from paper_2603_16428_b200.sharded import VocabShardedLCE
        sharded = VocabShardedLCE(V, budget_bytes=args.budget, schedule="R" if args.schedule == "R" else "S",
                                  emulate_shard=(G, 0) if G != g else None)
        assert (sharded.v0, sharded.v1) == (v0, v1)
        if sharded.schedule == "S":  # the workspace shares the budget with the module's dX buffers
            ws_budget = sharded.s_workspace_budget(N, H)
    native = multi and not dp and sharded.schedule == "S" and args.comm == "native"
    comm_note = None
    if native and G != g:
        # Timing only: rank 0 of G emulated GPUs through the native call, with a callback transport
        # that replicates this rank's statistics into all G slots and leaves the fp32 dX partial
        # as it is (no exchange; results are those of identical shards).
        class _Raw:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": "|u1",
                                                 "version": 3, "strides": None}

        def _ag(send, recv, nbytes, stream):
            src = torch.as_tensor(_Raw(send, nbytes), device=dev)
            torch.as_tensor(_Raw(recv, nbytes * G), device=dev).view(G, nbytes).copy_(src.expand(G, nbytes))

        comm = slf.Comm.callbacks(0, G, _ag, lambda buf, count, stream: None)
        comm_note = f"native, emulated rank 0 of {G} (statistics replicated, no exchange; timing only)"
    elif native:  # the library runs the whole sharded step, collectives included (slf_lce_fwd_bwd_sharded)
        try:
            comm = slf.Comm.from_process_group(device=local)
            if args.p2p_stats or args.p2p_dx:
                comm.set_p2p((1 if args.p2p_stats else 0) | (2 if args.p2p_dx else 0))
        except Exception as e:  # a transport that cannot start: same kernels, Python orchestration
            native = False
            comm_note = f"native communicator unavailable ({e}); torch.distributed orchestration"
            print(comm_note, file=sys.stderr)
    if native:
        ws = torch.empty(slf.sharded_workspace_bytes(N, H, V, G, 0 if G != g else rank, args.budget),
                         dtype=torch.uint8, device=dev)
    else:
        ws = slf.alloc_workspace(N_l, H, V_l, dev, schedule="S" if (multi and not dp and sharded.schedule == "S")
                                 else args.schedule, budget_bytes=ws_budget)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    dX = torch.empty(N_l, H, dtype=torch.bfloat16, device=dev)
    dW = torch.empty(V_l, H, dtype=torch.bfloat16, device=dev)
    extra = ws.numel()
    if dp:  # slf_lce_fwd_bwd_dp: global MEAN denominator, loss and dW syncs inside the library
        dp_comm = slf.Comm.from_process_group(device=local)
    elif multi and not native:
        if sharded.schedule == "S":
            C_s, _ = slf.s_plan(N, H, V_l, ws_budget)
            extra += 2 * C_s * H * 4 + (g + 1) * C_s * 16  # double-buffered fp32 dX partials + statistics
        else:
            extra += g * N * 16 + N * H * 4  # gathered statistics + fp32 dX partial

    def step(Xs=X, ts=t):
        if not multi:
            slf.lce_fwd_bwd(Xs, W, ts, out=(loss, dX, dW), workspace=ws, budget_bytes=args.budget,
                            schedule=args.schedule)
            return loss
        if dp:
            l, _, _ = slf.lce_fwd_bwd_dp(Xs, W, ts, dp_comm, sync_dweight=True, workspace=ws, out=(loss, dX, dW),
                                         budget_bytes=args.budget, schedule=args.schedule)
            return l
        if native:  # a P2P timeout poisons the loss; checked once after the timed region
            l, _, _ = slf.lce_fwd_bwd_sharded(Xs, W, ts, V, comm, workspace=ws, out=(loss, dX, dW),
                                              budget_bytes=args.budget, check_p2p=False)
            return l
        l, _, _ = sharded.forward_backward(Xs, W, ts, workspace=ws, dW_out=dW, dX_out=dX)
        return l

    def barrier():
        if multi:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid) if hasattr(
        torch.cuda.get_device_properties(dev), "uuid") else str(local)
    clocks = Clocks(uuid)
    with clocks:
        time.sleep(0.3)
        barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    # Per-step distribution (median and min): the same K steps again with an event
    # pair around each step (kept out of the timed region: an event between steps forfeits one
    # programmatic-dependent-launch overlap per step).
    barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a_, b_ in evs:
        a_.record(stream)
        step()
        b_.record(stream)
    torch.cuda.synchronize()
    per_step = np.array([a_.elapsed_time(b_) for a_, b_ in evs])
    # Per-kernel breakdown (roofline): the same K steps again with a CUDA-event pair around every
    # library launch.  Kept out of the timed region above because events between launches also
    # disable programmatic dependent launch.
    barrier()
    torch.cuda.synchronize()
    with slf.Profile() as prof:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    barrier()
    if multi:
        tt = torch.tensor([ms, *per_step.tolist()], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0].item())
        per_step = tt[1:].cpu().numpy()
    p2p_timeouts = comm.p2p_timeouts() if native and comm_note is None and (args.p2p_stats or args.p2p_dx) else 0
    if p2p_timeouts:
        raise RuntimeError(f"rank {rank}: a P2P exchange wait timed out during the benchmark")

    # End to end through the public API with HOST buffers: per step, the pinned host->device copy
    # of the step's inputs (hidden states, targets), the fused call and a device->host read of the
    # loss.  On one GPU this is the C-ABI host-input call (slf_lce_fwd_bwd_host: hidden rows are
    # copied chunk by chunk on a copy stream while earlier chunks compute); sharded runs copy with
    # torch and call their module.
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(inp.X[n0:n1].view(np.int16)).view(torch.bfloat16).pin_memory()
        th = torch.from_numpy(inp.t[n0:n1]).pin_memory()
        # Two staging sets and pinned loss slots: step k+1's input copy runs under step k, and step
        # k's loss is read on the host right after step k+1 is enqueued (every step's H2D copy and
        # loss D2H read are inside the timed region).
        lh = [torch.empty(1, dtype=torch.float32).pin_memory() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        Xd = torch.empty_like(X)
        td = torch.empty_like(t)
        stg = [slf.HostStaging(N_l, H, dev) for _ in range(2)] if not multi else None
        losses = []

        def e2e_step(i):
            k = i % 2
            if not multi:
                slf.lce_fwd_bwd_host(Xh, W, th, dX=dX, dW=dW, loss_host=lh[k], staging=stg[k], workspace=ws,
                                     budget_bytes=args.budget, schedule=args.schedule)
            else:
                Xd.copy_(Xh, non_blocking=True)
                td.copy_(th, non_blocking=True)
                lo = step(Xd, td)
                lh[k].copy_(lo.reshape(1), non_blocking=True)
            done[k].record(torch.cuda.current_stream(dev))
            if i > 0:  # the previous step's loss, read on the host
                done[1 - k].synchronize()
                losses.append(float(lh[1 - k][0]))

        def e2e_drain(i_last):
            done[i_last % 2].synchronize()
            losses.append(float(lh[i_last % 2][0]))

        for i in range(2):
            e2e_step(i)
        e2e_drain(1)
        barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for i in range(args.steps):
            e2e_step(i)
        e2e_drain(args.steps - 1)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / args.steps
        if multi:
            tt = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        assert all(np.isfinite(losses)) and len(losses) == args.steps + 2
        e2e = {"value": N / (ems / 1e3), "unit": UNIT, "ms_per_step": ems, "loss_read": "every step, one step late",
               "h2d_bytes_per_step": int(X.numel() * 2 + t.numel() * 4), "d2h_bytes_per_step": 4}

    if rank != 0:
        if multi:
            if native:
                comm.close()
            if dp and dp_comm is not None:
                dp_comm.close()
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    ck = clocks.summary(w0, w1)
    energy = None
    if ck.get("power_w_median"):  # the step is power-capped: energy per step is what the kernels trade
        energy = {"j_per_step": ck["power_w_median"] * ms / 1e3,
                  "tokens_per_joule": N / (ck["power_w_median"] * ms / 1e3) / g,
                  "note": "median board power (nvidia-smi power.draw samples inside the timed region) x device "
                          "time per step (per GPU)"}
    flops = 6.0 * N * H * V
    tflops = flops / (ms / 1e3) / 1e12
    kinds = prof.kinds
    launches = int(sum(v["launches"] for k, v in kinds.items() if not k.startswith("comm_")))  # our kernels only
    gemm_kinds = {k: v for k, v in kinds.items() if k.startswith("gemm")}
    dom_name, dom = max(gemm_kinds.items(), key=lambda kv: kv[1]["ms"])
    dom_ms_per_launch = dom["ms"] / dom["launches"]
    dom_flops_per_launch = dom["flops"] / dom["launches"]
    achieved = dom_flops_per_launch / (dom_ms_per_launch / 1e3) / 1e12
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_path):
        try:
            traffic = json.load(open(prof_path)).get(args.config, {}).get(dom_name)
        except Exception:
            traffic = None
    exec_flops = sum(v["flops"] for k, v in kinds.items() if k.startswith("gemm")) / args.steps
    kernels = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                   **({"tflops": v["flops"] / (v["ms"] / 1e3) / 1e12} if v["flops"] else {}),
                   **({"gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9} if v["bytes"] else {})}
               for k, v in kinds.items()}
    out = {
        "metric": METRIC, "value": N / (ms / 1e3), "unit": UNIT, "n_gpus": g, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        # the same N tokens of one call at every GPU count: strong scaling (dp: the batch split)
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "step_ms": {"mean_timed_region": ms, "median": float(np.median(per_step)), "min": float(per_step.min()),
                    "max": float(per_step.max()),
                    "note": "median/min/max from a second pass of K steps with an event pair per step"
                            + (" (max over ranks per step)" if multi else "")},
        "config": {"workload": f"{args.config} LM head N={N} H={H} V={V}", "N": N, "H": H, "V": V,
                   "V_per_gpu": V_l, "N_per_gpu": N_l,
                   "parallelism": (f"token-sharded data parallel x{g}" if dp else f"vocab-sharded x{g}")
                   if multi else "single GPU",
                   "targets": args.dist, "logit_std": args.alpha, "ignore_frac": 0.05,
                   "l2": "inputs larger than L2 (W alone is %.2f GB vs 126 MB L2); no flush" % (V_l * H * 2 / 1e9),
                   "plan": slf.sharded_plan_describe(N, H, V, G, 0 if G != g else rank, args.budget) if native else
                   slf.plan_describe(N_l, H, V_l, budget_bytes=ws_budget, schedule=args.schedule),
                   **({"comm": "native (slf_lce_fwd_bwd_dp, slf_comm NCCL)"} if dp else {}),
                   **({"comm": comm_note if (native and comm_note) else
                       ("native (slf_comm NCCL inside libslf_lce.so" + (", P2P statistics all-gather" if
                                args.p2p_stats else "") + (", P2P dX exchange kernel" if args.p2p_dx else "") + ")")
                       if native else
                       (comm_note or "torch.distributed NCCL (Python orchestration)")} if multi and not dp else {})},
        "tflops": tflops, "tflops_executed": exec_flops / (ms / 1e3) / 1e12,
        "frac_of_peak_burst": tflops / peaks["burst"],
        "frac_of_peak_sustained": tflops / peaks["sustained"],
        "frac_of_datasheet_dense_bf16": tflops / 2250.0,  # nominal 2.25 PF dense bf16 (unverified here)
        "roofline": {"bound": "tensor", "kernel": dom_name, "achieved": achieved, "peak": peaks["sustained"],
                     "unit": "TFLOP/s", "frac": achieved / peaks["sustained"], "traffic": traffic,
                     "peak_kind": "bf16 sustained (kernel timed inside a long step), " + peaks["source"],
                     "frac_of_burst": achieved / peaks["burst"],
                     # context: the sustained peak was measured at the peak run's median SM clock
                     # (nvidia-smi samples; under the power cap they lag the kernels' own clock, so no
                     # clock-normalised fraction is derived from them — DESIGN.md §7b uses in-kernel
                     # clock64 / globaltimer counters instead)
                     **({"clock_mhz_peak_run": peaks["sustained_mhz"], "clock_mhz_this_run": ck["sm_mhz"]}
                        if peaks.get("sustained_mhz") and ck.get("sm_mhz") else {}),
                     "ncu": "profiles/ncu_r02h.md (tensor pipe active % per kernel, DRAM bytes)"},
        "kernels": kernels,
        "comm": ({"allgather_ms_per_step": kinds.get("comm_allgather", {}).get("ms", 0.0) / args.steps,
                  "allreduce_ms_per_step": kinds.get("comm_allreduce", {}).get("ms", 0.0) / args.steps,
                  "collectives_per_step": sum(kinds.get(k, {}).get("launches", 0)
                                              for k in ("comm_allgather", "comm_allreduce")) / args.steps,
                  "note": "NCCL calls inside the library, CUDA events on the communicator's stream (rank 0; they "
                          "overlap the next chunk's GEMMs)"} if multi else None),
        "gpu_launches": launches,
        "memory": {"extra_device_bytes": int(extra), "logits_bytes_per_gpu": N_l * V_l * 2,
                   "frac_of_logits_per_gpu": extra / (N_l * V_l * 2), "frac_of_global_logits": extra / (N * V * 2),
                   "frac_of_spec_logits_and_grads": extra / (2 * N_l * V_l * 2)},  # SPEC's 2*N*V*2
        "clocks": ck,
        "energy": energy,
        "e2e": e2e,
    }
    if g == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(inp, args.config)
    print(json.dumps(out), file=json_out, flush=True)
    if multi:
        if native:
            comm.close()
        if dp and dp_comm is not None:
            dp_comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
