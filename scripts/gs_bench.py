"""Gram-Schmidt pass bandwidth on a GS-dominated Lanczos (diagonal operator, SURVEY §8d C5 style).

    python scripts/gs_bench.py [n] [m]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import json  # noqa: E402

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    ctx = d.Context(0)
    spec = 1.0 + (np.arange(n, dtype=np.float64) % 1000)
    op = d.diagonal_operator(ctx, spec)
    d.lanczos_distributed(ctx, 4, op, n, 1)  # warm-up
    ctx.set_option("ktimers_reset", 1)
    ctx.set_option("ktimers", 1)
    st = d.lanczos_distributed(ctx, m, op, n, 3)
    ctx.set_option("ktimers", 0)
    for k, (ms, cnt, work) in sorted(ctx.kernel_stats().items()):
        if k.startswith("gs_"):
            gbs = work / (ms / 1e3) / 1e9
            print(f"{k:10s} n={n} m={m} launches={cnt:.0f} {ms:9.2f} ms  {gbs:8.1f} GB/s  {gbs / hbm:6.3f} of HBM")
    print("iterations", st.iterations)
    ctx.close()


if __name__ == "__main__":
    main()
