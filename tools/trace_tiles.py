"""Per-tile timeline of one grouped GEMM launch (debug; not a bench line).

Runs the fused call twice on the Llama-8B head (schedule S by default) with SLF_DEBUG_TRACE set to
the group launch of chunk `--chunk` of the second call, then prints, for unit 0's leader CTA, the
per-tile MMA issue time, the MMA's wait for a free TMEM accumulator, the epilogue's wait for the
accumulator and its processing time, split by problem (0 = dX, 1 = dW for schedule S).

    python tools/trace_tiles.py [--schedule S] [--chunk 2]
"""
import argparse
import ctypes
import os
import sys

import numpy as np


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schedule", default="S")
    ap.add_argument("--chunk", type=int, default=2)
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--stats", action="store_true", help="trace the stash GEMM instead of the group")
    a = ap.parse_args()
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth
    c = synth.CONFIGS[a.config]
    N, H, V = c["N"], c["H"], c["V"]
    launches_per_call = None
    import torch
    import paper_2603_16428_b200 as slf
    from paper_2603_16428_b200._lib import lib
    desc = slf.plan_describe(N, H, V, schedule=a.schedule)
    kv = dict(x.split("=") for x in desc.split())
    assert kv["schedule"] == "S", "trace layout assumes schedule S (stash GEMM, group) per chunk"
    # chunk list of the fused call (extended chunks: slf_lce.cu phase_s; SLF_S_NO_EXT disables)
    C, ld = int(kv["row_chunk"]), (V + 7) // 8 * 8
    nch, r0, chunk_rows = 0, 0, []
    while r0 < N:
        rows = min(C, N - r0)
        if rows == C and not os.environ.get("SLF_S_NO_EXT"):
            e = min(max(0, (N - r0 - C) * H // (ld + H)), C) // 256 * 256
            rows += e
        r0 += rows
        nch += 1
        chunk_rows.append(rows)
    launches_per_call = 2 * nch
    target = launches_per_call + 2 * a.chunk + (0 if a.stats else 1)
    os.environ["SLF_DEBUG_TRACE"] = str(target)  # read once, at the first launch
    inp = synth.make_inputs(N, H, V, seed=0)
    X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
    W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda()
    t = torch.from_numpy(inp.t).cuda()
    ws = slf.alloc_workspace(N, H, V, X.device, schedule=a.schedule)
    for _ in range(2):
        slf.lce_fwd_bwd(X, W, t, workspace=ws, schedule=a.schedule)
    torch.cuda.synchronize()
    n = 1024 * 8
    buf = (ctypes.c_uint64 * n)()
    assert lib().slf_debug_trace_read(buf, n) == 0
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
    used = tr[:, 6] > 0
    tr = tr[used]
    t0 = tr[:, 0].min()
    print(f"{desc}\ntraced launch #{target} (group of chunk {a.chunk}); {len(tr)} tiles on unit 0")
    mma_wait = tr[:, 1] - tr[:, 0]
    mma_issue = tr[:, 2] - tr[:, 1]
    epi_wait = tr[:, 4] - tr[:, 3]
    epi_to_release = tr[:, 5] - tr[:, 4]
    epi_total = tr[:, 6] - tr[:, 4]
    rows = chunk_rows[a.chunk]
    kblocks = {0: (H if a.stats else V) / 64, 1: rows / 64}
    print(f"chunk rows {rows}; K-blocks per tile: {kblocks}")
    for p in sorted(set(tr[:, 7].tolist())):
        m = tr[:, 7] == p
        print(f"problem {p}: MMA issue per K-block {np.median(mma_issue[m]) / kblocks[p]:.0f} cyc (ideal 512)")
        print(f"problem {p}: {m.sum()} tiles | MMA issue (tile) median {np.median(mma_issue[m]):.0f} cyc, "
              f"MMA wait for free TMEM median {np.median(mma_wait[m]):.0f} (total {mma_wait[m].sum()}) | "
              f"epilogue wait for acc median {np.median(epi_wait[m]):.0f}, acc->release median "
              f"{np.median(epi_to_release[m]):.0f}, acc->end median {np.median(epi_total[m]):.0f}")
    span = tr[:, 6].max() - t0
    print(f"span {span} cycles; MMA waiting on TMEM {mma_wait.sum()} ({mma_wait.sum() / span:.1%}); "
          f"MMA issuing {mma_issue.sum()} ({mma_issue.sum() / span:.1%})")
    for i in range(min(12, len(tr))):
        print("tile", i, "prob", tr[i, 7], "rel stamps", (tr[i, :7] - t0).tolist())


if __name__ == "__main__":
    main()
