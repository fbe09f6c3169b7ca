"""One-off end-to-end parity at scale: the C3 workload (MLP 3072-2048-2048-10, n = 10,510,346,
C = 1, b = 512, curvature batch 512, k = 20, m = budget, AdamW) for one outer round of DHO2 (10 steps incl.
the refresh) on the GPU against the UNMODIFIED reference library's train() on identical data and seeds.

    python scripts/parity_c3_trajectory.py [outer_rounds] [base optimizer]     (the CPU side takes ~10 min per round)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from oracle.bindings import CpuChecker, base_cfg, blobs_dataset, reference_available, train_cfg  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    base = sys.argv[2] if len(sys.argv) > 2 else "adamw"
    sizes = [3072, 2048, 2048, 10]
    N, b, curv, k = 5120, 512, 512, 20
    R = CpuChecker("reference" if reference_available() else "port")
    X, y = blobs_dataset(N, 3072, 10, seed=7)
    w0 = R.mlp_init(sizes, 1)
    t0 = time.perf_counter()
    ref = R.train_mlp(train_cfg("dho2", base_cfg(base), k=k, l=0, outer_rounds=K, inner_epochs=1, batch_size=b,
                                curvature_batch=curv, seed=1), sizes, X, y, w0, workers=1, ncls=10)
    t_cpu = time.perf_counter() - t0
    ctx = d.Context(0)
    mlp = d.MlpOracle(ctx, sizes)
    cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig(base), k=k, l=0, outer_rounds=K, inner_epochs=1,
                          batch_size=b, curvature_batch=curv, seed=1)
    t0 = time.perf_counter()
    res = d.train(ctx, cfg, mlp, d.Dataset(X, y, 10, 7), w0, workers=1)
    t_gpu = time.perf_counter() - t0
    rel = np.linalg.norm(res.w_final - ref["w_final"]) / np.linalg.norm(ref["w_final"])
    print(f"C3 DHO2 ({base}) trajectory parity: n={len(w0)}, {K} outer round(s) x 10 steps; {R.kind} library "
          f"{R.max_threads()} threads {t_cpu:.0f} s vs GPU {t_gpu:.2f} s (incl. setup)")
    print(f"  epochs {list(res.epoch)} vs {list(ref['epoch'])}; refreshes {res.ese_refreshes} vs {ref['refreshes']}")
    print(f"  params rel-L2 {rel:.2e} (bar 1e-4); max-abs {np.abs(res.w_final - ref['w_final']).max():.2e}")
    print(f"  epoch loss GPU {res.loss} ref {ref['loss']} rel {np.abs(res.loss - ref['loss']) / np.abs(ref['loss'])}"
          f" (bar 1e-3 Adam-family)")
    print(f"  epoch accuracy GPU {res.acc} ref {ref['acc']}; ADMM residual GPU {res.residual_norm} ref {ref['resid']}")


if __name__ == "__main__":
    main()
