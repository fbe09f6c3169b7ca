"""Ritz-vector extraction bandwidth: tensor-core (3xTF32) vs CUDA-core kernel at n rows, m, k.

    python scripts/ritz_bench.py [n] [m] [k]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 80
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    ctx = d.Context(0)
    spec = 1.0 + (np.arange(n, dtype=np.float64) % 1000)
    op = d.diagonal_operator(ctx, spec)
    st = d.lanczos_distributed(ctx, m, op, n, 3)
    for tc in (1, 0, 1, 0):
        ctx.set_option("ritz_tc", tc)
        d.extract_ese_distributed(ctx, st, k, 0)
        ctx.set_option("ktimers_reset", 1)
        ctx.set_option("ktimers", 1)
        for _ in range(3):
            d.extract_ese_distributed(ctx, st, k, 0)
        ctx.set_option("ktimers", 0)
        for name, (ms, cnt, work) in sorted(ctx.kernel_stats().items()):
            if name.startswith("extract"):
                print(f"ritz_tc={tc} {name:16s} {ms / cnt * 1e3:10.1f} us  {work / (ms / 1e3) / 1e9 if work else 0:8.1f} GB/s")
    ctx.close()


if __name__ == "__main__":
    main()
