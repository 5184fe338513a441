"""Mainloop rate of the tcgen05 core per operand layout (debug GEMM, fp32 epilogue amortised over
K = 16384; 592 pair tiles = 8 waves of 74 units).  Not a bench line.

    python tools/layout_rate.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16428_b200 as slf  # noqa: E402


def main():
    M, N, K = 256 * 37, 4096, 16384
    dev = "cuda"
    for a_mn in (0, 1):
        for b_mn in (0, 1):
            A = torch.randn(K, M, device=dev).to(torch.bfloat16) if a_mn else torch.randn(M, K, device=dev).to(torch.bfloat16)
            B = torch.randn(K, N, device=dev).to(torch.bfloat16) if b_mn else torch.randn(N, K, device=dev).to(torch.bfloat16)
            for _ in range(2):
                slf.debug_gemm(A, B, a_mn, b_mn, M, N, K)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                slf.debug_gemm(A, B, a_mn, b_mn, M, N, K)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"a_mn={a_mn} b_mn={b_mn}: {ms:.3f} ms {2.0 * M * N * K / ms / 1e9:.0f} TF/s")
            del A, B


if __name__ == "__main__":
    main()
