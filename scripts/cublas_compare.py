"""Calibration: our split-BF16x3 tcgen05 GEMM (3 bf16 products per output) against cuBLAS doing the same
three bf16 products as plain GEMMs (torch.matmul, bf16 in / fp32 accumulate), on the C4 shapes.

    python scripts/cublas_compare.py
cuBLAS is a measuring stick here only; it is never on the library's path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from paper_2505_00982_b200.api import test_gemm  # noqa: E402

SHAPES = [(1024, 3584, 7168, "HVP R-forward / R-backward (B=1024)"), (3584, 3584, 2048, "HVP weight block"),
          (8192, 3584, 3584, "gradient forward (8192)"), (3584, 3584, 8192, "gradient weight block")]


def cublas_ms(M, N, K, reps=10):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps * 3):  # three products per split-BF16x3 output
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def ours_ms(ctx, M, N, K, reps=5):
    rng = np.random.default_rng(0)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    test_gemm(ctx, A, B, 0)
    ctx.set_option("ktimers_reset", 1)
    ctx.set_option("ktimers", 1)
    for _ in range(reps):
        test_gemm(ctx, A, B, 0)
    ctx.set_option("ktimers", 0)
    st = ctx.kernel_stats()
    ms = sum(v[0] for k, v in st.items() if k.startswith("gemm3"))
    cnt = sum(v[1] for k, v in st.items() if k.startswith("gemm3"))
    return ms / cnt


def main():
    ctx = d.Context(0)
    for M, N, K, what in SHAPES:
        c = cublas_ms(M, N, K)
        o = ours_ms(ctx, M, N, K)
        fl = 2.0 * M * N * K
        print(f"{what:36s} M={M:5d} N={N:5d} K={K:5d}: cuBLAS 3 x bf16 {c * 1e3:8.1f} us ({3 * fl / (c / 1e3) / 1e12:6.0f} TF/s)"
              f"  ours split-BF16x3 {o * 1e3:8.1f} us ({3 * fl / (o / 1e3) / 1e12:6.0f} TF/s issued)  ratio {c / o:5.2f}")
    ctx.close()


if __name__ == "__main__":
    main()
