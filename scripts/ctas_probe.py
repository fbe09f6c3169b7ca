import sys, os, time
sys.path.insert(0, '/root/repo'); os.chdir(os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import numpy as np
import paper_2505_00982_b200 as d
from oracle.bindings import blobs_dataset
ctx = d.Context(0)
sizes = [784, 256, 10]
X, y = blobs_dataset(128, 784, 10, seed=7)
mlp = d.MlpOracle(ctx, sizes)
w = mlp.init_params(1)
op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
n = len(w)
for cps in (1, 2):
    ctx.set_option("mlp_small_ctas_per_sm", cps)
    for fused in (1, 0):
        ctx.set_option("lanczos_small", fused)
        for _ in range(2):
            d.lanczos_distributed(ctx, 40, op, n, 11).close()
        ctx.set_option("ktimers_reset", 1); ctx.set_option("ktimers", 1)
        st = d.lanczos_distributed(ctx, 40, op, n, 11)
        ctx.synchronize(); ctx.set_option("ktimers", 0)
        ks = ctx.kernel_stats()
        print(cps, fused, {k: round(v[0] * 1e3 / max(v[1], 1), 1) for k, v in ks.items()}, st.tridiag.diag[:3])
        st.close()
