"""cuBLAS (torch.matmul) on the GEMM shapes of one schedule-S chunk at the Llama-8B head, for
context against the fused kernels (not a bench line).  Times with CUDA events, back to back.

    python tools/cublas_shapes.py [--rows 1152]
"""
import argparse

import torch


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1152)
    a = ap.parse_args()
    C, H, V = a.rows, 4096, 128256
    dev = "cuda"
    X = torch.randn(C, H, device=dev, dtype=torch.bfloat16)
    W = torch.randn(V, H, device=dev, dtype=torch.bfloat16) * 0.02
    G = torch.randn(C, V, device=dev, dtype=torch.bfloat16) * 1e-3
    dW = torch.zeros(V, H, device=dev, dtype=torch.bfloat16)
    out_z = torch.empty(C, V, device=dev, dtype=torch.bfloat16)
    out_dx = torch.empty(C, H, device=dev, dtype=torch.bfloat16)
    fl = 2.0 * C * H * V
    for name, fn in (
        ("logits  Z = X W^T      ", lambda: torch.matmul(X, W.t(), out=out_z)),
        ("dX      G W            ", lambda: torch.matmul(G, W, out=out_dx)),
        ("dW      G^T X (store)  ", lambda: torch.matmul(G.t(), X, out=dW)),
        ("dW      G^T X (+= bf16)", lambda: dW.addmm_(G.t(), X)),
    ):
        ms = timeit(fn)
        print(f"rows={C} {name} {ms:.3f} ms  {fl / ms / 1e9:.0f} TF/s")
    big = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    ms = timeit(lambda: torch.matmul(big, big), 50)
    print(f"8192^3 square {ms:.3f} ms {2 * 8192 ** 3 / ms / 1e9:.0f} TF/s")


if __name__ == "__main__":
    main()
