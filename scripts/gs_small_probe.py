"""Per-kernel breakdown of the launch-per-step Gram-Schmidt at small n (C5 cells, diagonal operator).

    python scripts/gs_small_probe.py [n] [m]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_00982_b200 as d

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_250_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ctx = d.Context(0)
spec = 1.0 + (np.arange(n, dtype=np.float64) % 1000)
op = d.diagonal_operator(ctx, spec)
ctx.set_option("lanczos_small", 0)
d.lanczos_distributed(ctx, m, op, n, 1).close()
ctx.set_option("ktimers_reset", 1); ctx.set_option("ktimers", 1)
st = d.lanczos_distributed(ctx, m, op, n, 3)
ctx.synchronize(); ctx.set_option("ktimers", 0)
for k, (ms, cnt, work) in sorted(ctx.kernel_stats().items(), key=lambda kv: -kv[1][0]):
    print(f"{k:24s} {cnt:5.0f} {ms:8.3f} ms  avg {ms / max(cnt, 1) * 1e3:8.1f} us  {work / (ms / 1e3) / 1e9 if work else 0:8.1f} GB/s")
import time
for _ in range(2):
    ctx.synchronize(); t = time.perf_counter()
    st2 = d.lanczos_distributed(ctx, m, op, n, 3); ctx.synchronize()
    print(f"whole refresh (graph, untimed kernels): {(time.perf_counter() - t) * 1e3:.3f} ms wall, iters {st2.iterations}")
    st2.close()
