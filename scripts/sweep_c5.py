"""C5 microbench sweep at G = 1 (BASELINE.json configs[4]): Lanczos on the diagonal
QuadraticOracle operator (GS-dominated) over n x k (m = 4k), and the C4-family MLP HVP over the hidden
width H (B = 1024). Cells whose basis + V_hat + 12 vectors exceed 178 GB are skipped.

    python scripts/sweep_c5.py [--quick]
Prints one line per cell: refresh ms, Gram-Schmidt GB/s (fraction of the measured HBM peak), HVP ms and
useful / issued tensor TF/s."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    j = json.load(open(p)) if os.path.exists(p) else {}
    return j.get("hbm_gbs", 6650.0), j.get("bf16_tflops_sustained", 1400.0)


def lanczos_cell(ctx, n, k, hbm):
    m = 4 * k
    need = 4.0 * (m + 1 + k + 12) * n
    if need > 178e9:
        return f"lanczos n={n:>11,d} k={k:>3d} m={m:>3d}: skipped ({need / 1e9:.0f} GB > 178 GB)"
    spec = 1.0 + (np.arange(n, dtype=np.float64) % 1000)
    op = d.diagonal_operator(ctx, spec)
    del spec
    d.lanczos_distributed(ctx, 2, op, n, 1)  # warm-up / allocation
    ctx.set_option("ktimers_reset", 1)
    ctx.set_option("ktimers", 1)
    ctx.mark(0)
    st = d.lanczos_distributed(ctx, m, op, n, 3)
    ese = d.extract_ese_distributed(ctx, st, min(k, st.iterations), 0)
    ctx.mark(1)
    ctx.set_option("ktimers", 0)
    ms = ctx.elapsed_ms(0, 1)
    ks = ctx.kernel_stats()
    # (fused refresh: the whole recurrence is one launch, "lanczos_small"; its time includes the O(n) HVPs)
    gs_ms = sum(v[0] for kk, v in ks.items() if kk.startswith("gs_") or kk == "lanczos_small")
    gs_b = sum(v[2] for kk, v in ks.items() if kk.startswith("gs_") or kk == "lanczos_small")
    rz = ks.get("extract.ritz", (0.0, 0, 0.0))
    tq = ks.get("extract.tql2", (0.0, 0, 0.0))
    ese.close()
    st.close()
    op.close()
    gbs = gs_b / (gs_ms / 1e3) / 1e9
    return (f"lanczos n={n:>11,d} k={k:>3d} m={m:>3d}: refresh {ms:9.1f} ms  GS {gs_ms:9.1f} ms {gbs:7.0f} GB/s "
            f"({gbs / hbm:.2f} of HBM)  ritz {rz[0]:7.1f} ms  eig {tq[0]:6.1f} ms")


def hvp_cell(ctx, H, tf_peak):
    sizes = [3072] + [H] * 8 + [10]
    mlp = d.MlpOracle(ctx, sizes)
    n = mlp.dim()
    w = mlp.init_params(1)
    X, y = d.blobs_dataset(1024, 3072, 10, seed=7)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
    d.lanczos_distributed(ctx, 2, op, n, 1)
    ctx.set_option("ktimers_reset", 1)
    ctx.set_option("ktimers", 1)
    st = d.lanczos_distributed(ctx, 6, op, n, 3)
    ctx.set_option("ktimers", 0)
    ks = ctx.kernel_stats()
    g_ms = sum(v[0] for kk, v in ks.items() if kk.startswith("gemm3"))
    g_fl = sum(v[2] for kk, v in ks.items() if kk.startswith("gemm3"))
    tf = g_fl / (g_ms / 1e3) / 1e12
    per_hvp = st.iterations and (sum(v[0] for kk, v in ks.items() if not kk.startswith("gs_") and not kk.startswith("phase"))
                                 / st.iterations)
    st.close()
    op.close()
    mlp.close()
    return (f"hvp  H={H:>5d} n={n:>11,d} B=1024: {per_hvp:8.2f} ms/HVP (kernels)  GEMM {tf:6.1f} TF/s useful "
            f"({tf / tf_peak:.2f}), {3 * tf:6.1f} issued ({3 * tf / tf_peak:.2f} of bf16 sustained)")


def main():
    quick = "--quick" in sys.argv
    hbm, tfp = peaks()
    ctx = d.Context(0)
    ctx.set_option("graphs", 0)
    t0 = time.time()
    ns = [1_250_000, 10_500_000, 101_000_000] + ([] if quick else [408_800_000])
    for n in ns:
        for k in (8, 32, 128):
            print(lanczos_cell(ctx, n, k, hbm), flush=True)
    for H in ([256, 1024, 3584] + ([] if quick else [7424])):
        print(hvp_cell(ctx, H, tfp), flush=True)
    print(f"# sweep wall {time.time() - t0:.0f} s", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
