"""Tridiagonal eigensolve time: split (QL chain + shared-memory rotation replay + selection) vs the
single-CTA tql2 kernel, at the Lanczos sizes m of C1-C5.

    python scripts/tql2_bench.py [m ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402


def main():
    ms_list = [int(a) for a in sys.argv[1:]] or [40, 80, 128, 256, 512, 1000]
    ctx = d.Context(0)
    for m in ms_list:
        n = max(20_000, 40 * m)
        spec = 1.0 + np.sin(np.arange(n) * 0.731) * 3.0 + 0.01 * (np.arange(n) % 97)
        op = d.diagonal_operator(ctx, spec)
        st = d.lanczos_distributed(ctx, m, op, n, 3)
        k = min(32, st.iterations)
        res = {}
        for split in (1, 0, 1, 0):
            ctx.set_option("tql2_split", split)
            d.extract_ese_distributed(ctx, st, k, 0)
            ctx.set_option("ktimers_reset", 1)
            ctx.set_option("ktimers", 1)
            for _ in range(3):
                d.extract_ese_distributed(ctx, st, k, 0)
            ctx.set_option("ktimers", 0)
            ks = ctx.kernel_stats()
            ms, cnt, _ = ks["extract.tql2"]
            res[split] = ms / cnt
            if split:
                parts = "  ".join(f"{kk} {v[0] / v[1]:.3f}" for kk, v in sorted(ks.items()) if kk.startswith("eig."))
        ctx.set_option("tql2_split", 1)
        print(f"tql2 m={st.iterations:5d}: single-CTA {res[0]:8.3f} ms   split {res[1]:8.3f} ms   "
              f"({res[0] / res[1]:.1f}x)   [{parts}]", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
