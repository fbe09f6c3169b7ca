"""One rank's share of the C4 step at G = 1, 2, 4, 8 GPUs, measured on ONE B200.

A PROJECTION, not a multi-GPU measurement: each component of one rank's work is timed on this GPU at the
size that rank would run (SURVEY §8e partitioning), and the collectives are added from their byte counts at
an ASSUMED NVLink 5 bus bandwidth:
  gradient     C/G logical workers x b samples, full model                  (trainer.cpp:92-103)
  HVP          B/G curvature samples, full model (batch-split HVP)          (dist_lanczos.cpp:79)
  Gram-Schmidt ceil(n/G) rows, m = 80, full reorthogonalisation              (dist_lanczos.cpp:55-119)
  update       ceil(n/G) rows, r = 32, AdamW                                 (optimizer.cpp:81-129)
  collectives  per Lanczos iteration all_gather(v) + reduce_scatter(hv), n floats each; per step
               reduce_scatter(g) + all_gather(w_a), n floats each; small all-reduces ignored
Per-kernel device times come from the library's CUDA-event timers (serialised kernels). Also reports the
HVP GEMMs' issued tensor fraction at M = B/G (the verdict's question: does M = 128 at G = 8 collapse?).

    python scripts/rank_share.py [--busbw 700] [--gs 1]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from bench import CONFIGS, hvp_flops, grad_flops, mlp_dim  # noqa: E402


def ktimed(ctx, fn):
    ctx.set_option("ktimers_reset", 1)
    ctx.set_option("ktimers", 1)
    fn()
    ctx.synchronize()
    ctx.set_option("ktimers", 0)
    return ctx.kernel_stats()


def total_ms(stats, pred=lambda k: True):
    return sum(ms for k, (ms, cnt, w) in stats.items() if pred(k) and not k.startswith("phase."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--busbw", type=float, default=700.0, help="assumed NCCL bus bandwidth per GPU, GB/s")
    ap.add_argument("--gs", type=int, default=1, help="also time the GS passes at n/G rows")
    args = ap.parse_args()
    c = CONFIGS["c4"]
    sizes, C, b, B, k, m = c["sizes"], c["workers"], c["b"], c["curv"], c["k"], c["m"]
    n = mlp_dim(sizes)
    peak_tf = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops_sustained", 1377.9) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1377.9
    ctx = d.Context(0)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    X, y = d.blobs_dataset(C * b, sizes[0], sizes[-1], seed=7)
    rounds = 10  # refresh every P * rounds_per_epoch = 10 steps (C4)
    print(f"# C4 one-rank share on one B200: n={n}, C={C} x b={b}, B={B}, m={m}, k={k}; "
          f"collectives at an assumed {args.busbw:.0f} GB/s bus bandwidth (projection)")
    for G in (1, 2, 4, 8):
        rows = -(-n // G)
        # gradient of this rank's C/G workers
        gb = d.Batch(X[: C * b // G], y[: C * b // G], sizes[-1])
        mlp.grad(w, gb)
        st = ktimed(ctx, lambda: mlp.grad(w, gb))
        t_grad = total_ms(st)
        # HVPs on B/G samples: a 4-iteration Lanczos on the MLP operator, GEMM + packing kernels only
        op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X[: B // G], y[: B // G], sizes[-1]))
        d.lanczos_distributed(ctx, 2, op, n, 1)
        st = ktimed(ctx, lambda: d.lanczos_distributed(ctx, 4, op, n, 1))
        hvp_keys = lambda kk: not kk.startswith(("gs_", "lz_", "lanczos", "eig", "extract"))  # noqa: E731
        t_hvp = total_ms(st, hvp_keys) / 4
        gemm_ms = total_ms(st, lambda kk: kk.startswith("gemm3")) / 4
        issued = 3 * hvp_flops(sizes, B // G) / (gemm_ms / 1e3) / 1e12 / peak_tf if gemm_ms > 0 else 0.0
        op.close()
        # GS at n/G rows, m iterations (diagonal operator: the passes alone)
        t_gs = None
        if args.gs:
            spec = 1.0 + (np.arange(rows) % 1000).astype(np.float64)
            dop = d.diagonal_operator(ctx, spec)
            d.lanczos_distributed(ctx, 2, dop, rows, 1)
            st = ktimed(ctx, lambda: d.lanczos_distributed(ctx, m, dop, rows, 3))
            t_gs = total_ms(st, lambda kk: kk.startswith("gs_"))
            dop.close()
        # update pass on n/G rows, r = 32 (device kernels only)
        V = np.zeros((rows, k))
        V[np.arange(k) * (rows // k), np.arange(k)] = 1.0
        ese = d.EseResult.from_host(ctx, np.linspace(40, 1, k), V)
        opt = d.BaseOptimizer(ctx, d.BaseConfig("adamw"), rows)
        gg = np.random.default_rng(0).standard_normal(rows)
        d.admm_deltas(gg, gg, ese, opt, gg, 0.1, 1e-2)
        st = ktimed(ctx, lambda: d.admm_deltas(gg, gg, ese, opt, gg, 0.1, 1e-2))
        t_upd = total_ms(st, lambda kk: kk.startswith("upd_"))
        ese.close()
        opt.close()
        del V
        # collectives (n floats each; a ring moves (G-1)/G of it per GPU)
        coll = 0.0 if G == 1 else (G - 1) / G * 4.0 * n / (args.busbw * 1e9) * 1e3
        t_refresh = m * (t_hvp + 2 * coll) + (t_gs or 0.0)
        t_step = t_grad + t_upd + 2 * coll + t_refresh / rounds
        print(f"G={G}: grad {t_grad:7.2f} ms  hvp {t_hvp:6.2f} ms/iter (GEMM issued {issued:.2f} of sustained at "
              f"M={B // G})  gs {t_gs if t_gs is not None else float('nan'):7.1f} ms/refresh  update {t_upd:5.2f} ms  "
              f"collective {coll:5.2f} ms each -> refresh {t_refresh:7.1f} ms, step {t_step:6.2f} ms, "
              f"{1e3 / t_step:6.2f} steps/s per job (projection)", flush=True)


if __name__ == "__main__":
    main()
