"""Times the small-model path's passes on the device (C1/C2 shapes) — used for ncu captures."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_00982_b200 as d
from oracle.bindings import blobs_dataset

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = d.Context(0)
sizes = [784, 256, 10]
X, y = blobs_dataset(max(B, 128), 784, 10, seed=7)
mlp = d.MlpOracle(ctx, sizes)
w = mlp.init_params(1)
op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X[:B], y[:B], 10))
n = len(w)
for _ in range(2):
    st = d.lanczos_distributed(ctx, 40, op, n, 11)
    st.close()
t0 = time.time()
for _ in range(reps):
    st = d.lanczos_distributed(ctx, 40, op, n, 11)
    st.close()
ctx.synchronize()
print(f"B={B}: lanczos m=40 {1e3 * (time.time() - t0) / reps:.3f} ms/refresh (host wall, eager)")
ctx.set_option("ktimers_reset", 1)
ctx.set_option("ktimers", 1)
st = d.lanczos_distributed(ctx, 40, op, n, 11)
ctx.synchronize()
ctx.set_option("ktimers", 0)
for k, v in sorted(ctx.kernel_stats().items()):
    print(f"  {k}: {v[0]:.3f} ms / {int(v[1])} = {1e3 * v[0] / max(v[1], 1):.1f} us")
