"""C1/C2-shaped update (n = 203,530, r = 10): the fused small-n update vs the three-pass path."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_00982_b200 as d
ctx = d.Context(0)
n, r = 203_530, 10
rng = np.random.default_rng(0)
V = np.linalg.qr(rng.standard_normal((n, r)))[0]
ese = d.EseResult.from_host(ctx, np.linspace(40, 1, r), V)
g = rng.standard_normal(n)
outs = {}
for small in (1, 0):
    ctx.set_option("upd_small", small)
    opt = d.BaseOptimizer(ctx, d.BaseConfig("adam"), n)
    for _ in range(3):
        res = d.admm_deltas(g, g * 0.1, ese, opt, g * 0.01, 0.1, 1e-2)
    ctx.set_option("ktimers_reset", 1); ctx.set_option("ktimers", 1)
    for _ in range(5):
        res = d.admm_deltas(g, g * 0.1, ese, opt, g * 0.01, 0.1, 1e-2)
    ctx.synchronize(); ctx.set_option("ktimers", 0)
    ks = ctx.kernel_stats()
    print(small, {k: round(v[0] * 1e3 / max(v[1], 1), 1) for k, v in ks.items() if k.startswith("upd")})
    outs[small] = res
    opt.close()
a, b = outs[1], outs[0]
for name in ("newton", "base"):
    x, y = getattr(a, name), getattr(b, name)
    print(name, float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300)))
