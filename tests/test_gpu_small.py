"""The small-model path (csrc/mlp_small.cu): each MLP pass of a small model (HVP <= ctx option
mlp_small_mflop, default 2 GFLOP: the C1/C2 784-256-10 models) is ONE cooperative persistent launch on the
CUDA cores instead of the tcgen05 GEMM sequence. Parity against the CPU checker (oracle.cpp:451-687 restated)
and the tensor-core path, determinism, graph capture of the cooperative launch, and the refresh / trainer
paths through it."""
import numpy as np
import pytest

import paper_2505_00982_b200 as d

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def kernels_of(ctx, fn):
    ctx.set_option("ktimers_reset", 1)
    ctx.set_option("ktimers", 1)
    try:
        out = fn()
        ctx.synchronize()
    finally:
        ctx.set_option("ktimers", 0)
    return out, ctx.kernel_stats()


CASES = [([784, 256, 10], 128, "tanh", "softmax_ce", 10), ([784, 256, 10], 512, "relu", "softmax_ce", 10),
         ([20, 16, 12, 5], 37, "tanh", "mse", 5), ([13, 24, 1], 1, "tanh", "mse", 0),
         ([64, 96, 96, 96, 10], 200, "relu", "mse", 10), ([33, 70, 41, 7], 65, "tanh", "softmax_ce", 7),
         ([5, 2, 3], 300, "tanh", "softmax_ce", 3),
         ([20, 16, 40], 50, "tanh", "mse", 40),            # output wider than a tile: separate output phase
         ([30, 40, 33], 70, "relu", "softmax_ce", 33),
         ([12] + [9] * 7 + [4], 45, "tanh", "softmax_ce", 4),  # L = 8, the deepest small-path model
         ([3000, 24, 10], 64, "relu", "softmax_ce", 10)]   # long K (input 3000) on the first layer


@pytest.mark.parametrize("sizes,B,act,loss,ncls", CASES)
def test_small_path_vs_checker_and_tensor_path(ctx, port, sizes, B, act, loss, ncls):
    from oracle.bindings import blobs_dataset
    X, y = blobs_dataset(B, sizes[0], max(ncls, 1), seed=21)
    if ncls == 0:
        y = np.cos(np.arange(B) * 0.21)
    a, lo = {"tanh": 0, "relu": 1}[act], {"softmax_ce": 0, "mse": 1}[loss]
    w = port.mlp_init(sizes, 4)
    w = w + 0.05 * port.rng_normal(3, len(w))
    v = port.rng_normal(8, len(w))
    b = d.Batch(X, y, ncls)
    mlp = d.MlpOracle(ctx, sizes, act, loss)
    (hv, g, val), ks = kernels_of(ctx, lambda: (mlp.hvp(w, v, b), mlp.grad(w, b), mlp.value(w, b)))
    assert "mlp_small.hvp" in ks and "mlp_small.grad" in ks and "mlp_small.prep" in ks
    assert not any(k.startswith("gemm3") for k in ks)  # no tensor-core GEMM on this path
    hv_ref = port.mlp_hvp(sizes, w, v, X, y, ncls, a, lo)
    g_ref = port.mlp_grad(sizes, w, X, y, ncls, a, lo)
    val_ref = port.mlp_value(sizes, w, X, y, ncls, a, lo)
    # fp32 products and sums of fp32 operands: relative L2 <= 1e-5 (measured ~1e-7 .. 1e-6)
    assert rel_l2(hv, hv_ref) < 1e-5
    assert rel_l2(g, g_ref) < 1e-5
    assert abs(val - val_ref) <= 1e-6 * max(1.0, abs(val_ref))
    if ncls:
        assert abs(mlp.accuracy(w, b) - port.mlp_accuracy(sizes, w, X, y, ncls, a, lo)) <= 1.5 / B
    # bitwise repeatable (fixed split order)
    assert (mlp.hvp(w, v, b) == hv).all() and (mlp.grad(w, b) == g).all()
    # the tensor-core path on the same inputs
    ctx.set_option("mlp_small", 0)
    try:
        (hv_t, g_t), ks_t = kernels_of(ctx, lambda: (mlp.hvp(w, v, b), mlp.grad(w, b)))
    finally:
        ctx.set_option("mlp_small", 1)
    assert not any(k.startswith("mlp_small") for k in ks_t)
    assert rel_l2(hv_t, hv) < 1e-4 and rel_l2(g_t, g) < 1e-4
    mlp.close()


def test_small_path_depth_limit(ctx, port):
    """Models deeper than the small path supports (L > 8) take the tensor-core path, with the same results."""
    from oracle.bindings import blobs_dataset
    sizes = [12] + [9] * 8 + [4]
    X, y = blobs_dataset(40, 12, 4, seed=5)
    mlp = d.MlpOracle(ctx, sizes)
    w = port.mlp_init(sizes, 2)
    v = port.rng_normal(4, len(w))
    b = d.Batch(X, y, 4)
    (hv, g), ks = kernels_of(ctx, lambda: (mlp.hvp(w, v, b), mlp.grad(w, b)))
    assert not any(k.startswith("mlp_small") for k in ks)
    assert rel_l2(hv, port.mlp_hvp(sizes, w, v, X, y, 4, 0, 0)) < 1e-4
    assert rel_l2(g, port.mlp_grad(sizes, w, X, y, 4, 0, 0)) < 1e-4
    mlp.close()


def test_small_path_threshold(ctx):
    """Eligibility follows the HVP flop count at the call's batch size: above mlp_small_mflop the
    tensor-core path runs."""
    from oracle.bindings import blobs_dataset
    sizes = [784, 256, 10]
    X, y = blobs_dataset(512, 784, 10, seed=2)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    b = d.Batch(X, y, 10)
    ctx.set_option("mlp_small_mflop", 300.0)  # B = 512: 1.05 GFLOP > 300 MFLOP; B = 64: 131 MFLOP
    try:
        _, ks = kernels_of(ctx, lambda: mlp.grad(w, b))
        assert "mlp_small.grad" not in ks and any(k.startswith("gemm3") for k in ks)
        _, ks = kernels_of(ctx, lambda: mlp.grad(w, d.Batch(X[:64], y[:64], 10)))
        assert "mlp_small.grad" in ks
    finally:
        ctx.set_option("mlp_small_mflop", 2000.0)
    mlp.close()


def test_small_path_refresh_c1_vs_checker(ctx, port):
    """A C1 refresh (784-256-10, curvature batch 128, m = 40, k = 10) through the small path: eigenvalues and
    B against the checker's refresh (§8d bars), and bitwise repeatable."""
    from oracle.bindings import blobs_dataset
    sizes, B, m, k = [784, 256, 10], 128, 40, 10
    X, y = blobs_dataset(B, 784, 10, seed=7)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
    n = len(w)
    runs = []
    for _ in range(2):
        (st, ese), ks = kernels_of(ctx, lambda: (lambda s_: (s_, d.extract_ese_distributed(ctx, s_, k, 0)))(
            d.lanczos_distributed(ctx, m, op, n, 11)))
        assert "lanczos_small" in ks  # the fused refresh: one launch for the m iterations
        runs.append((st.tridiag.diag.copy(), st.tridiag.offdiag.copy(), ese.eigvals.copy()))
        ese.close()
        st.close()
    assert all((x == y_).all() for x, y_ in zip(runs[1], runs[0]))
    ref = port.lanczos(dict(kind=2, n=n, sizes=sizes, w=w, X=X, y=y, ncls=10), m, 11, k=k, want_basis=False)
    diag, off, ev = runs[0]
    hn = float(np.max(np.abs(ref["eigvals"])))
    assert np.max(np.abs(ev - ref["eigvals"]) / np.abs(ref["eigvals"])) <= 1e-4
    assert np.max(np.abs(diag - ref["diag"])) <= 1e-5 * hn and np.max(np.abs(off - ref["off"])) <= 1e-5 * hn
    # the unfused small path (one launch per HVP, the GS kernels of lanczos.cu) agrees
    ctx.set_option("lanczos_small", 0)
    try:
        (st, ese), ks = kernels_of(ctx, lambda: (lambda s_: (s_, d.extract_ese_distributed(ctx, s_, k, 0)))(
            d.lanczos_distributed(ctx, m, op, n, 11)))
    finally:
        ctx.set_option("lanczos_small", 1)
    assert ks["mlp_small.hvp"][1] == m and "lanczos_small" not in ks
    assert np.max(np.abs(st.tridiag.diag - diag)) <= 1e-6 * hn
    assert np.max(np.abs(ese.eigvals - ev) / np.abs(ev)) <= 1e-6
    ese.close()
    st.close()
    op.close()
    mlp.close()


@pytest.mark.parametrize("recurrence,safeguard", [(1, 1), (0, 1), (1, 0)])
def test_fused_refresh_matches_unfused(ctx, port, recurrence, safeguard):
    """The fused refresh (one persistent launch) against the launch-per-step path on the same operator, both
    projection modes and with / without the reference's reorthogonalisation safeguard; a tanh MSE model with
    a rapidly decaying spectrum so that safeguard passes and a breakdown-free long run both occur."""
    from oracle.bindings import blobs_dataset
    sizes, B, m = [40, 64, 32, 3], 96, 60
    X, y = blobs_dataset(B, 40, 3, seed=9)
    mlp = d.MlpOracle(ctx, sizes, "tanh", "mse")
    w = mlp.init_params(2)
    n = len(w)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 3))
    out = []
    ctx.set_option("lanczos_recurrence", recurrence)
    try:
        for fused in (1, 0):
            ctx.set_option("lanczos_small", fused)
            opts = d.DistLanczosOptions(d.LanczosOptions(reorth_safeguard=bool(safeguard)))
            st = d.lanczos_distributed(ctx, m, op, n, 5, opts)
            out.append((st.iterations, st.breakdown, st.tridiag.diag.copy(), st.tridiag.offdiag.copy(),
                        st.safeguard_passes))
            st.close()
    finally:
        ctx.set_option("lanczos_small", 1)
        ctx.set_option("lanczos_recurrence", 1)
    (i1, b1, d1, o1, s1), (i0, b0, d0, o0, s0) = out
    print(f"fused: iterations {i1} breakdown {b1} safeguard passes {s1}; unfused: {i0} {b0} {s0}")
    assert i1 == i0 and b1 == b0
    assert abs(s1 - s0) <= max(1, s0 // 10)  # safeguard triggers sit on a threshold: rounding may move one
    hn = float(np.max(np.abs(d0[:i0]))) + float(np.max(np.abs(o0[:i0])))
    k = min(i0, 20)  # the first iterations agree closely; later ones follow the (fp32) loss of orthogonality
    assert np.max(np.abs(d1[:k] - d0[:k])) <= 1e-5 * hn and np.max(np.abs(o1[:k] - o0[:k])) <= 1e-5 * hn
    op.close()
    mlp.close()


def test_small_path_trainer_graph_bitwise(ctx):
    """The trainer's refresh graph with the small path's cooperative launches as kernel nodes (C2-shaped
    model and workers): bitwise the eager run, and the graph was replayed."""
    from oracle.bindings import blobs_dataset
    sizes = [784, 256, 10]
    X, y = blobs_dataset(1280, 784, 10, seed=3)
    probe = d.MlpOracle(ctx, sizes)
    w0 = probe.init_params(2)
    _, ks = kernels_of(ctx, lambda: probe.grad(w0, d.Batch(X[:128], y[:128], 10)))
    assert "mlp_small.grad" in ks
    probe.close()
    out = []
    g0 = ctx.stat("lanczos_graph_launches")
    for graphs in (0, 1):
        ctx.set_option("graphs", graphs)
        try:
            mlp = d.MlpOracle(ctx, sizes)
            cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("momentum"), k=10, l=0, outer_rounds=3,
                                  inner_epochs=1, epochs=1, batch_size=32, curvature_batch=128, seed=5)
            out.append(d.train(ctx, cfg, mlp, d.Dataset(X, y, 10, 7), w0, workers=4))
            mlp.close()
        finally:
            ctx.set_option("graphs", 1)
    assert out[0].ese_refreshes == out[1].ese_refreshes == 3
    assert (out[0].w_final == out[1].w_final).all()
    assert (out[0].loss == out[1].loss).all()
    assert ctx.stat("lanczos_graph_launches") - g0 >= 1


@pytest.mark.parametrize("n,m", [(1_200_000, 24), (1000, 30)])
def test_fused_refresh_diagonal_operator(ctx, n, m):
    """The fused refresh on a diagonal operator (lanczos_small = 2; several row tiles per CTA slice at
    n = 1.2 M) against the launch-per-step path, and the identity operator's breakdown after one step."""
    spec = 1.0 + (np.arange(n, dtype=np.float64) % 97) * 0.37
    op = d.diagonal_operator(ctx, spec)
    out = []
    try:
        for fused in (2, 0):
            ctx.set_option("lanczos_small", fused)
            st = d.lanczos_distributed(ctx, m, op, n, 7)
            out.append((st.iterations, st.breakdown, st.tridiag.diag.copy(), st.tridiag.offdiag.copy()))
            st.close()
        (i1, b1, d1, o1), (i0, b0, d0, o0) = out
        assert i1 == i0 and b1 == b0
        k = min(i0, 12)
        assert np.max(np.abs(d1[:k] - d0[:k])) <= 1e-5 * spec.max()
        assert np.max(np.abs(o1[:k] - o0[:k])) <= 1e-5 * spec.max()
        ident = d.diagonal_operator(ctx, np.ones(n))
        ctx.set_option("lanczos_small", 2)
        st = d.lanczos_distributed(ctx, m, ident, n, 7)
        assert st.breakdown and st.iterations == 1 and abs(st.tridiag.diag[0] - 1.0) < 1e-6
        st.close()
        ident.close()
    finally:
        ctx.set_option("lanczos_small", 1)
    op.close()
