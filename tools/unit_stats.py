"""Per-unit (CTA pair) MMA feed counters of one GEMM launch (debug; not a bench line): cycles per
K-block, and the shares of the MMA issuer's time spent waiting for a loaded stage (operand feed)
or for a free accumulator (epilogue), and the producer's wait for a free stage.

    python tools/unit_stats.py --what debug|stats|group [--chunk 2]
"""
import argparse
import ctypes
import os
import sys

import numpy as np


def chunk_list(N, H, V, C):
    ld, r0, out = (V + 7) // 8 * 8, 0, []
    while r0 < N:
        rows = min(C, N - r0)
        if rows == C and not os.environ.get("SLF_S_NO_EXT"):
            rows += min(max(0, (N - r0 - C) * H // (ld + H)), C) // 256 * 256
        out.append(rows)
        r0 += rows
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="debug")
    ap.add_argument("--chunk", type=int, default=2)
    ap.add_argument("--mn", default="00", help="debug GEMM: a_mn b_mn (e.g. 11: both operands MN-major)")
    a = ap.parse_args()
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    if a.what == "debug":
        os.environ["SLF_DEBUG_TRACE"] = "3"
    else:
        import synth
        c = synth.CONFIGS["llama8b"]
        N, H, V = c["N"], c["H"], c["V"]
        import paper_2603_16428_b200 as slf0
        kv = dict(x.split("=") for x in slf0.plan_describe(N, H, V, schedule="S").split())
        nch = len(chunk_list(N, H, V, int(kv["row_chunk"])))
        os.environ["SLF_DEBUG_TRACE"] = str(2 * nch + 2 * a.chunk + (0 if a.what == "stats" else 1))
    import torch
    import paper_2603_16428_b200 as slf
    import paper_2603_16428_b200._lib as L
    if os.environ.get("SLF_SO"):  # experiment builds (tools/exp)
        L.SO_PATH = os.environ["SLF_SO"]
    from paper_2603_16428_b200._lib import lib
    if a.what == "debug":
        M, N_, K = 256 * 37, 4096, 16384
        am, bm = int(a.mn[0]), int(a.mn[1])
        A = torch.randn(K if am else M, M if am else K, device="cuda").to(torch.bfloat16)
        B = torch.randn(K if bm else N_, N_ if bm else K, device="cuda").to(torch.bfloat16)
        for _ in range(5):
            slf.debug_gemm(A, B, am, bm, M, N_, K)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            slf.debug_gemm(A, B, am, bm, M, N_, K)
        e1.record()
        torch.cuda.synchronize()
        print(f"debug GEMM {e0.elapsed_time(e1) / 20:.3f} ms per launch (events)")
    else:
        inp = synth.make_inputs(N, H, V, seed=0)
        X = torch.from_numpy(inp.X.view(np.int16)).view(torch.bfloat16).cuda()
        W = torch.from_numpy(inp.W.view(np.int16)).view(torch.bfloat16).cuda()
        t = torch.from_numpy(inp.t).cuda()
        ws = slf.alloc_workspace(N, H, V, X.device, schedule="S")
        for _ in range(2):
            slf.lce_fwd_bwd(X, W, t, workspace=ws, schedule="S")
    torch.cuda.synchronize()
    n = (1024 + 256) * 8
    buf = (ctypes.c_uint64 * n)()
    assert lib().slf_debug_trace_read(buf, n) == 0
    u = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)[1024:].astype(np.int64)
    u = u[u[:, 4] > 0]
    span = u[:, 3] - u[:, 2]
    kb = u[:, 4]
    cpk = span / kb
    fw = u[:, 0] / span
    tw = u[:, 1] / span
    ew = u[:, 5] / span
    ghz = span / np.maximum(u[:, 7], 1)
    print(f"in-kernel SM clock (clock64 / globaltimer) median {np.median(ghz):.3f} GHz; MMA span median "
          f"{np.median(u[:, 7]) / 1e6:.3f} ms")
    print(f"{a.what}: {len(u)} units, tiles/unit {np.median(u[:, 6]):.0f}, K-blocks/unit {np.median(kb):.0f}")
    for name, x in (("cycles per K-block", cpk), ("MMA wait full (feed)", fw), ("MMA wait TMEM (epilogue)", tw),
                    ("producer wait empty", ew)):
        q = np.percentile(x, [0, 10, 50, 90, 100])
        print(f"  {name:26s} min {q[0]:.3f} p10 {q[1]:.3f} med {q[2]:.3f} p90 {q[3]:.3f} max {q[4]:.3f}")
    order = np.argsort(cpk)
    print("  slowest units:", [(int(i), round(float(cpk[i]))) for i in order[-6:]])
    print("  fastest units:", [(int(i), round(float(cpk[i]))) for i in order[:6]])
    # load balance: each unit's MMA span (first to last issue) and work
    ns = u[:, 7].astype(np.float64)
    q = np.percentile(ns / 1e6, [0, 50, 100])
    print(f"  unit MMA span ms           min {q[0]:.3f} med {q[1]:.3f} max {q[2]:.3f}")
    by_span = np.argsort(ns)
    print("  longest units (unit, span ms, tiles, K-blocks):",
          [(int(i), round(float(ns[i]) / 1e6, 3), int(u[i, 6]), int(kb[i])) for i in by_span[-5:]])
    print("  shortest units (unit, span ms, tiles, K-blocks):",
          [(int(i), round(float(ns[i]) / 1e6, 3), int(u[i, 6]), int(kb[i])) for i in by_span[:5]])


if __name__ == "__main__":
    main()
