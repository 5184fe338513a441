"""Sustained (3 s) rate, SM clock and board power of the tcgen05 core (debug GEMM) against cuBLAS
(torch.matmul) on comparable bf16 GEMMs — is a gap per clock or per joule?  Not a bench line.

    python tools/power_compare.py
"""
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16428_b200 as slf  # noqa: E402


def sustained(fn, flops, secs=3.0):
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    samples, stop = [], threading.Event()

    def sampler():
        time.sleep(0.8)
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.05)

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    th = threading.Thread(target=sampler)
    th.start()
    n, t0 = 0, time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    clk = sorted(s[0] for s in samples)[len(samples) // 2]
    pw = sorted(s[1] for s in samples)[len(samples) // 2]
    tf = flops / ms / 1e9
    return f"{ms:.3f} ms {tf:.0f} TF/s  sm {clk} MHz  {pw:.0f} W  {tf / pw:.2f} TF/J  {tf / clk * 1e3 / 148 / 2:.0f} flop/clk/SM (of 8192)"


def main():
    dev = "cuda"
    M, N, K = 256 * 37, 4096, 16384
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    B = torch.randn(N, K, device=dev).to(torch.bfloat16)
    print("tcgen05 core K-major  ", sustained(lambda: slf.debug_gemm(A, B, 0, 0, M, N, K), 2.0 * M * N * K))
    D = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    print("cuBLAS same shape bf16", sustained(lambda: torch.matmul(A, B.t(), out=D), 2.0 * M * N * K))
    S = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    O = torch.empty_like(S)
    print("cuBLAS 8192^3         ", sustained(lambda: torch.matmul(S, S, out=O), 2.0 * 8192 ** 3))


if __name__ == "__main__":
    main()
