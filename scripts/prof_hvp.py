"""Small, profiler-friendly workload: C4-shaped HVPs (and optionally gradients) on one GPU.

    python scripts/prof_hvp.py [--config c4] [--m 3] [--grad 1]

Runs a Lanczos refresh with m iterations on the C4 model (prepare + m cached HVPs + GS passes), then
`--grad` gradient evaluations at the C4 global batch, printing per-kernel device times. Used for
`ncu` captures (a full bench.py run launches ~15k kernels)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--m", type=int, default=3)
    ap.add_argument("--grad", type=int, default=0)
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--cta", type=int, default=0, help="0 auto, 1 single-CTA, 2 CTA pair")
    ap.add_argument("--ab", type=int, default=0, help="A/B rounds alternating --abopt values (GEMM rows only)")
    ap.add_argument("--abopt", default="gemm_cta", help="context option to alternate in the A/B rounds")
    ap.add_argument("--abvals", default="1,2", help="comma-separated values of --abopt")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    ctx = d.Context(0)
    ctx.set_option("gemm_splits", args.splits)
    mlp = d.MlpOracle(ctx, c["sizes"])
    w = mlp.init_params(1)
    X, y = d.blobs_dataset(max(c["curv"], c["b"] * c["workers"]), c["sizes"][0], c["sizes"][-1], seed=7)
    ctx.set_option("gemm_cta", args.cta)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X[: c["curv"]], y[: c["curv"]], c["sizes"][-1]))
    gb = d.Batch(X[: c["b"] * c["workers"]], y[: c["b"] * c["workers"]], c["sizes"][-1])

    def run(tag, gemm_only):
        ctx.set_option("ktimers_reset", 1)
        ctx.set_option("ktimers", 1)
        st = d.lanczos_distributed(ctx, args.m, op, mlp.dim(), 7)
        ese = d.extract_ese_distributed(ctx, st, min(4, st.iterations), 0)
        for _ in range(args.grad):
            mlp.grad(w, gb)
        ctx.synchronize()
        ctx.set_option("ktimers", 0)
        print(tag, "ritz values", ese.eigvals)
        for k, (ms, cnt, work) in sorted(ctx.kernel_stats().items(), key=lambda kv: -kv[1][0]):
            if gemm_only and not k.startswith("gemm"):
                continue
            tf = work / (ms / 1e3) / 1e12 if ms > 0 and k.startswith("gemm") else 0.0
            print(f"{tag} {k:40s} {cnt:6.0f} {ms:10.3f} ms  avg {ms / max(cnt, 1) * 1e3:9.1f} us  {tf:7.1f} TF/s")

    if args.ab:
        run("warm", True)
        for r in range(args.ab):
            for val in [int(x) for x in args.abvals.split(",")]:
                ctx.set_option(args.abopt, val)
                run(f"r{r}/{args.abopt}={val}", True)
    else:
        run("", False)
    ctx.close()


if __name__ == "__main__":
    main()
