"""C5 small-n Lanczos cells (diagonal operator) through the fused refresh and the launch-per-step path."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_00982_b200 as d
import json
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6468.0)
ctx = d.Context(0)
for n in (1_250_000, 4_000_000, 10_500_000):
    spec = 1.0 + (np.arange(n, dtype=np.float64) % 1000)
    op = d.diagonal_operator(ctx, spec)
    for k in (8, 32):
        m = 4 * k
        for fused in (1, 0):
            ctx.set_option("lanczos_small", 2 if fused else 0)
            ctx.set_option("lanczos_small_max_n", 2e7)
            d.lanczos_distributed(ctx, m, op, n, 1).close()
            ctx.set_option("ktimers_reset", 1); ctx.set_option("ktimers", 1)
            st = d.lanczos_distributed(ctx, m, op, n, 3)
            ctx.synchronize(); ctx.set_option("ktimers", 0)
            ks = ctx.kernel_stats()
            gs = [(kk, v) for kk, v in ks.items() if kk.startswith("gs_") or kk == "lanczos_small"]
            ms = sum(v[0] for _, v in gs); b = sum(v[2] for _, v in gs)
            print(f"n={n:>10,d} k={k:>3d} m={m:>3d} fused={fused}: GS(+HVP) {ms:7.2f} ms {b / ms / 1e6:7.0f} GB/s ({b / ms / 1e6 / hbm:.2f} of HBM) iters {st.iterations} diag0 {st.tridiag.diag[0]:.6f}", flush=True)
            st.close()
    op.close()
