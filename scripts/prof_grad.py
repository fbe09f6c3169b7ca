"""One C4 mean-gradient evaluation (8192 samples) — a short workload for ncu captures of the big GEMMs.

    python scripts/prof_grad.py [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_00982_b200 as d  # noqa: E402
from bench import CONFIGS  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    c = CONFIGS["c4"]
    ctx = d.Context(0)
    mlp = d.MlpOracle(ctx, c["sizes"])
    w = mlp.init_params(1)
    B = c["b"] * c["workers"]
    X, y = d.blobs_dataset(B, c["sizes"][0], c["sizes"][-1], seed=7)
    b = d.Batch(X, y, c["sizes"][-1])
    for _ in range(reps):
        mlp.grad(w, b)
    ctx.synchronize()
    ctx.close()


if __name__ == "__main__":
    main()
