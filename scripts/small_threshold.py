"""Where the small-model path stops paying: per-HVP device time (kernel timers, eager, inside a 6-iteration
Lanczos) of the small path (one launch per HVP) and the tcgen05 GEMM path, over models around the
mlp_small_mflop threshold."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_00982_b200 as d
from oracle.bindings import blobs_dataset

ctx = d.Context(0)
ctx.set_option("lanczos_small", 0)
ctx.set_option("mlp_small_mflop", 1e9)  # eligibility decided by the mlp_small switch alone
for sizes, B in [([784, 256, 10], 128), ([784, 256, 10], 512), ([784, 512, 10], 512), ([784, 1024, 10], 512),
                 ([1024, 1024, 1024, 10], 256), ([1024, 1024, 1024, 10], 512), ([2048, 2048, 10], 512),
                 ([3072, 2048, 2048, 10], 512)]:
    X, y = blobs_dataset(B, sizes[0], 10, seed=1)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    n = mlp.dim()
    fl = 2.0 * B * sum((5 + 3 * (t > 0)) * sizes[t] * sizes[t + 1] for t in range(len(sizes) - 1))
    res = {}
    for small in (1, 0):
        ctx.set_option("mlp_small", small)
        op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
        d.lanczos_distributed(ctx, 3, op, n, 1).close()
        ctx.set_option("ktimers_reset", 1); ctx.set_option("ktimers", 1)
        st = d.lanczos_distributed(ctx, 6, op, n, 1)
        ctx.synchronize(); ctx.set_option("ktimers", 0)
        ks = ctx.kernel_stats()
        hvp_ms = sum(v[0] for k, v in ks.items() if not k.startswith(("gs_", "lz_", "lanczos", "eig", "extract", "phase.")))
        res[small] = hvp_ms / 6 * 1e3
        st.close(); op.close()
    print(f"{str(sizes):28s} B={B:4d} HVP {fl / 1e9:6.2f} GFLOP: small {res[1]:8.1f} us  tcgen05 {res[0]:8.1f} us", flush=True)
    mlp.close()
