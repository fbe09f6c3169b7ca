"""Update-pass bandwidth (P1/P2/P3 of the fused FOSI/ADMM split update) at rank r, n rows.

    python scripts/upd_bench.py [n] [r] [staged variants, e.g. 0,5]
Times both P2 variants (bulk-copy staged / register-staged) with the kernel timers."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
    r = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    ctx = d.Context(0)
    rng = np.random.default_rng(0)
    V = rng.standard_normal((n, r)) / np.sqrt(n)
    ev = np.linspace(40.0, -3.0, r)
    ese = d.EseResult.from_host(ctx, ev, V)
    del V
    g, pi, w = rng.standard_normal(n), rng.standard_normal(n), rng.standard_normal(n)
    if len(sys.argv) > 3:  # explicit staged-variant list, e.g. "5" or "0,5"
        variants = [(1, int(v)) for v in sys.argv[3].split(",")]
    else:
        variants = [(1, v) for v in (0, 1, 5)] + [(0, 0)] + [(1, v) for v in (0, 1, 5)]
    for staged, var in variants:
        ctx.set_option("upd_p2_staged", staged)
        ctx.set_option("upd_p2_variant", var)
        opt = d.BaseOptimizer(ctx, d.BaseConfig("adamw", lr=1e-3), n)
        d.admm_deltas(g, pi, ese, opt, w, 0.3, 0.05)  # warm-up
        ctx.set_option("ktimers_reset", 1)
        ctx.set_option("ktimers", 1)
        for _ in range(3):
            d.admm_deltas(g, pi, ese, opt, w, 0.3, 0.05)
        ctx.set_option("ktimers", 0)
        for k, (ms, cnt, work) in sorted(ctx.kernel_stats().items()):
            if k.startswith("upd_"):
                print(f"staged={staged} var={var} {k} n={n} r={r} {ms / cnt * 1e3:9.1f} us  {work / (ms / 1e3) / 1e9:8.1f} GB/s")
    ctx.close()


if __name__ == "__main__":
    main()
