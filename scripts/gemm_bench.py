"""Times the split-BF16x3 tcgen05 GEMM (store epilogue) on the C4 shapes through the test hook.

    python scripts/gemm_bench.py [splits] [cta: 0 auto, 1 single-CTA, 2 CTA pair]
Reports per-launch device time (CUDA events) and useful / issued TFLOP/s."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from paper_2505_00982_b200.api import test_gemm  # noqa: E402

SHAPES = [  # (M, N, K, what)
    (1024, 3584, 7168, "HVP RZ/RU (B=1024, 2*3584)"),
    (1024, 3584, 3584, "HVP Z/U"),
    (3584, 3584, 2048, "HVP weight block (K=2B)"),
    (8192, 3584, 3584, "grad Z/U (B=8192)"),
    (3584, 3584, 8192, "grad weight block"),
]


def main():
    ctx = d.Context(0)
    splits = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    ctx.set_option("gemm_splits", splits)
    ctx.set_option("gemm_cta", cta)
    print("gemm_splits", splits, "gemm_cta", cta)
    rng = np.random.default_rng(0)
    for M, N, K, what in SHAPES:
        A = rng.standard_normal((M, K)).astype(np.float32)
        B = rng.standard_normal((N, K)).astype(np.float32)
        test_gemm(ctx, A, B, 0)  # warm-up
        ctx.set_option("ktimers_reset", 1)
        ctx.set_option("ktimers", 1)
        for _ in range(5):
            test_gemm(ctx, A, B, 0)
        ctx.set_option("ktimers", 0)
        st = ctx.kernel_stats()
        ms = sum(v[0] for k, v in st.items() if k.startswith("gemm3"))
        cnt = sum(v[1] for k, v in st.items() if k.startswith("gemm3"))
        per = ms / cnt
        tf = 2.0 * M * N * K / (per / 1e3) / 1e12
        print(f"{what:32s} M={M:5d} N={N:5d} K={K:5d}  {per * 1e3:8.1f} us  useful {tf:6.1f} TF/s  issued {3 * tf:6.1f}")
    ctx.close()


if __name__ == "__main__":
    main()
