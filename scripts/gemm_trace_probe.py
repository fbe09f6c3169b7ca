"""Per-CTA timeline of one R-forward (or R-backward) pair-GEMM launch inside a C4 refresh (test hook
dho2g_test_gemm_trace; %globaltimer). Investigation only.

    python scripts/gemm_trace_probe.py [fwd|bwd|store]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from paper_2505_00982_b200 import _lib  # noqa: E402
from bench import CONFIGS  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
c = CONFIGS["c4"]
ctx = d.Context(0)
mlp = d.MlpOracle(ctx, c["sizes"])
w = mlp.init_params(1)
X, y = d.blobs_dataset(c["curv"], c["sizes"][0], c["sizes"][-1], seed=7)
op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, c["sizes"][-1]))
d.lanczos_distributed(ctx, 2, op, mlp.dim(), 7).close()
n = 148
buf = (C.c_uint64 * (n * 8))()
for rep in range(2):
    _lib.lib.dho2g_test_gemm_trace(ctx.h, {"fwd": 3, "bwd": 4, "store": 5}[which], None, n)
    d.lanczos_distributed(ctx, 2, op, mlp.dim(), 7).close()
    _lib.lib.dho2g_test_gemm_trace(ctx.h, 0, buf, n)
    t = np.array(buf[:], dtype=np.float64).reshape(n, 8)
    live = t[:, 0] > 0
    t0 = t[live, 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)[live]
    names = ["start", "last MMA", "last acc ready", "end", "fixup done", "head epi done"]
    print(f"[{which} R-GEMM, rep {rep}] CTAs {live.sum()}: " + "  ".join(
        f"{nm} {np.nanmin(rel[:, i]):.1f}/{np.nanmedian(rel[:, i]):.1f}/{np.nanmax(rel[:, i]):.1f}"
        for i, nm in enumerate(names) if np.isfinite(rel[:, i]).any()))
    ep = rel[:, 5] - rel[:, 4]
    fx = rel[:, 4] - rel[:, 2]
    print(f"   head epilogue us (min/median/max): {np.nanmin(ep):.1f}/{np.nanmedian(ep):.1f}/{np.nanmax(ep):.1f};"
          f" fix-up wait: {np.nanmin(fx):.1f}/{np.nanmedian(fx):.1f}/{np.nanmax(fx):.1f};"
          f" last MMA -> end: {np.nanmedian(rel[:, 3] - rel[:, 1]):.1f}")
    a, b = t[live, 6] / 1e3, t[live, 7] / 1e3
    if a.max() > 0:
        print(f"   warp 4 per-tile sums (debug build): loads+TMEM+partials {np.median(a):.1f} us, block math+stores {np.median(b):.1f} us")
ctx.close()
