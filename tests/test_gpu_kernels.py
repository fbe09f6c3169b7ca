"""GPU parity of the individual sm_100a kernels against the CPU checker (oracle/) and exact fp64.

Tolerances: the device path is fp32 with split-BF16x3 tensor-core GEMMs and fp64
reductions, the checker is fp64. Each bound is written next to its assertion."""
import numpy as np
import pytest

import paper_2505_00982_b200 as d
from paper_2505_00982_b200.api import test_gemm as run_gemm

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


# ------------------------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (37, 10, 20), (130, 250, 200), (256, 384, 1000), (8, 3584, 7168),
                                   (1024, 256, 784), (300, 129, 65)])
def test_gemm3_tcgen05_vs_exact(ctx, M, N, K):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    tc = run_gemm(ctx, A, B, 0)
    st = run_gemm(ctx, A, B, 1)
    # split-BF16x3 drops lo*lo (2^-16 relative per product) -> bound 2e-5 of sum |a||b|
    assert np.max(np.abs(tc - exact) / scale) < 2e-5
    assert np.max(np.abs(st - exact) / scale) < 2e-5
    # the tensor-core and CUDA-core paths compute the same split products
    assert np.max(np.abs(tc - st) / scale) < 5e-6


@pytest.mark.parametrize("splits", [1, 2, 3, 4])
def test_gemm3_split_k_deterministic(ctx, splits):
    """Persistent tcgen05 GEMM with split-K: fixed-order combine -> bitwise repeatable, exact to 2e-5."""
    rng = np.random.default_rng(splits)
    A = rng.standard_normal((1024, 2048)).astype(np.float32)
    B = rng.standard_normal((640, 2048)).astype(np.float32)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    ctx.set_option("gemm_splits", splits)
    try:
        c1 = run_gemm(ctx, A, B, 0)
        c2 = run_gemm(ctx, A, B, 0)
    finally:
        ctx.set_option("gemm_splits", 0)
    assert (c1 == c2).all()
    assert np.max(np.abs(c1 - exact) / scale) < 2e-5


@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (300, 129, 65), (512, 3585, 256), (1024, 272, 7168),
                                   (2048, 1000, 3000), (1000, 16, 4096), (8, 40, 96)])
@pytest.mark.parametrize("cta", [1, 2])
def test_gemm3_cta_modes(ctx, M, N, K, cta):
    """Single-CTA (128x128, split-K) and CTA-pair (cta_group::2, 256x256, stream-K) kernels: exact to
    2e-5 of sum |a||b|, and the pair kernel's fixed-order stream-K combine is bitwise repeatable."""
    rng = np.random.default_rng(M + 11 * N + 3 * K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    ctx.set_option("gemm_cta", cta)
    try:
        c1 = run_gemm(ctx, A, B, 0)
        c2 = run_gemm(ctx, A, B, 0)
    finally:
        ctx.set_option("gemm_cta", 0)
    assert (c1 == c2).all()
    assert np.max(np.abs(c1 - exact) / scale) < 2e-5


@pytest.mark.parametrize("M,N,K", [(4096, 4096, 256), (6000, 2500, 300), (1024, 3584, 512), (8192, 768, 96)])
@pytest.mark.parametrize("dp", [0, 1])
def test_gemm3_pair_dp_stream_k(ctx, M, N, K, dp):
    """CTA-pair kernel schedule: data-parallel waves of whole tiles, then stream-K over the remainder
    (dp = 0: stream-K over everything). Exact to 2e-5 of sum |a||b| and bitwise repeatable."""
    rng = np.random.default_rng(M + N + K + dp)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    ctx.set_option("gemm_cta", 2)
    ctx.set_option("gemm_dp", dp)
    try:
        c1 = run_gemm(ctx, A, B, 0)
        c2 = run_gemm(ctx, A, B, 0)
    finally:
        ctx.set_option("gemm_cta", 0)
        ctx.set_option("gemm_dp", 1)
    assert (c1 == c2).all()
    assert np.max(np.abs(c1 - exact) / scale) < 2e-5


@pytest.mark.parametrize("M,N,K", [(1024, 3584, 2048), (512, 2048, 4096), (768, 1000, 3000), (1000, 2500, 1536)])
@pytest.mark.parametrize("group", [0, 1])
def test_gemm3_pair_groups(ctx, M, N, K, group):
    """CTA-pair kernel with few m-tiles: m-tile groups of pairs walking the same (n, k) ranges (group = 1,
    one pair per m-tile, stream-K fix-up between groups) against plain stream-K (group = 0). Exact to
    2e-5 of sum |a||b| and bitwise repeatable (ragged M and N included)."""
    rng = np.random.default_rng(M + 3 * N + 7 * K + group)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    ctx.set_option("gemm_cta", 2)
    ctx.set_option("gemm_group", group)
    try:
        c1 = run_gemm(ctx, A, B, 0)
        c2 = run_gemm(ctx, A, B, 0)
    finally:
        ctx.set_option("gemm_cta", 0)
        ctx.set_option("gemm_group", 1)
    assert (c1 == c2).all()
    assert np.max(np.abs(c1 - exact) / scale) < 2e-5


@pytest.mark.parametrize("M,N,K0,K1", [(256, 384, 130, 0), (300, 200, 100, 70), (700, 260, 64, 200),
                                       (1024, 512, 1024, 1024)])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("cta", [1, 2])
def test_gemm3_segmented_operands(ctx, M, N, K0, K1, a_mn, b_mn, cta):
    """K-major / MN-major operand windows with a two-segment K range (the MLP's [x | rx] contractions):
    C = A0 B0^T + A1 B1^T exact to 2e-5 of sum |a||b|; tcgen05 and CUDA-core paths agree."""
    from paper_2505_00982_b200.api import test_gemm_seg
    rng = np.random.default_rng(M + N + K0 + 7 * K1 + 3 * a_mn + b_mn)
    A0, B0 = rng.standard_normal((M, K0)), rng.standard_normal((N, K0))
    A1, B1 = rng.standard_normal((M, K1)), rng.standard_normal((N, K1))
    exact = A0 @ B0.T + A1 @ B1.T
    scale = np.abs(A0) @ np.abs(B0).T + np.abs(A1) @ np.abs(B1).T
    ctx.set_option("gemm_cta", cta)
    try:
        c = test_gemm_seg(ctx, A0, B0, A1, B1, 0, a_mn, b_mn)
    finally:
        ctx.set_option("gemm_cta", 0)
    s = test_gemm_seg(ctx, A0, B0, A1, B1, 1, a_mn, b_mn)
    assert np.max(np.abs(c - exact) / scale) < 2e-5
    assert np.max(np.abs(s - exact) / scale) < 2e-5


# ------------------------------------------------------------------------------------ MLP oracle
CASES = [([20, 16, 12, 5], 37, "tanh", "softmax_ce", 5), ([20, 16, 12, 5], 37, "relu", "softmax_ce", 5),
         ([20, 16, 12, 5], 37, "tanh", "mse", 5), ([13, 24, 1], 19, "tanh", "mse", 0),
         ([784, 256, 10], 128, "tanh", "softmax_ce", 10), ([64, 96, 96, 96, 10], 200, "tanh", "softmax_ce", 10)]


@pytest.fixture(params=[0, 1], ids=["tensor", "small"])
def mlp_path(ctx, request):
    """MLP tests below run on the tcgen05 GEMM path (mlp_small = 0) and the small-model path."""
    ctx.set_option("mlp_small", request.param)
    yield request.param
    ctx.set_option("mlp_small", 1)


@pytest.mark.parametrize("sizes,B,act,loss,ncls", CASES)
def test_mlp_oracle_vs_checker(ctx, port, sizes, B, act, loss, ncls, mlp_path):
    from oracle.bindings import blobs_dataset
    X, y = blobs_dataset(B, sizes[0], max(ncls, 1), seed=11)
    if ncls == 0:
        y = np.sin(np.arange(B) * 0.37)
    mlp = d.MlpOracle(ctx, sizes, act, loss)
    w = mlp.init_params(3)
    assert (w == port.mlp_init(sizes, 3)).all()  # oracle.cpp:386-394 bitwise on the host
    w = w + 0.05 * port.rng_normal(5, len(w))
    v = port.rng_normal(6, len(w))
    batch = d.Batch(X, y, ncls)
    a, lo = {"tanh": 0, "relu": 1}[act], {"softmax_ce": 0, "mse": 1}[loss]
    hv_ref = port.mlp_hvp(sizes, w, v, X, y, ncls, a, lo)
    g_ref = port.mlp_grad(sizes, w, X, y, ncls, a, lo)
    hv = mlp.hvp(w, v, batch)
    g = mlp.grad(w, batch)
    # fp32 + split-BF16x3: relative L2 <= 1e-4 (survey probe: ~4e-6)
    assert rel_l2(hv, hv_ref) < 1e-4
    assert rel_l2(g, g_ref) < 1e-4
    assert abs(mlp.value(w, batch) - port.mlp_value(sizes, w, X, y, ncls, a, lo)) <= 1e-5 * max(
        1.0, abs(port.mlp_value(sizes, w, X, y, ncls, a, lo)))
    if ncls:
        assert abs(mlp.accuracy(w, batch) - port.mlp_accuracy(sizes, w, X, y, ncls, a, lo)) <= 1.5 / B
    else:
        assert mlp.accuracy(w, batch) is None


@pytest.mark.parametrize("act,loss,xscale", [("tanh", "softmax_ce", 1e-3), ("relu", "mse", 1e-4), ("relu", "softmax_ce", 300.0),
                                             ("relu", "softmax_ce", 1e4)])
def test_mlp_scaled_fp16_operands_any_magnitude(ctx, port, act, loss, xscale):
    """Scaled-fp16 operand pairs (option gemm_f16) take each buffer's scale from the max of the values it holds:
    inputs 1e-4 .. 1e4, relu activations (unbounded) and MSE deltas stay within the fp32 tolerance of the
    checker, and agree with the bf16-pair path."""
    from oracle.bindings import blobs_dataset
    sizes, ncls = [24, 32, 16, 6], 6
    X, y = blobs_dataset(50, 24, ncls, seed=13)
    X = X * xscale
    a, lo = {"tanh": 0, "relu": 1}[act], {"softmax_ce": 0, "mse": 1}[loss]
    w = port.mlp_init(sizes, 5)
    v = port.rng_normal(17, len(w))
    hv_ref = port.mlp_hvp(sizes, w, v, X, y, ncls, a, lo)
    g_ref = port.mlp_grad(sizes, w, X, y, ncls, a, lo)
    out = {}
    for f16 in (1, 0):
        ctx.set_option("gemm_f16", f16)
        ctx.set_option("mlp_small", 0)  # the tensor-core operand formats
        try:
            mlp = d.MlpOracle(ctx, sizes, act, loss)
            b = d.Batch(X, y, ncls)
            out[f16] = (mlp.hvp(w, v, b), mlp.grad(w, b))
            mlp.close()
        finally:
            ctx.set_option("gemm_f16", 1)
            ctx.set_option("mlp_small", 1)
        assert np.isfinite(out[f16][0]).all() and np.isfinite(out[f16][1]).all()
        assert rel_l2(out[f16][0], hv_ref) < 1e-4 and rel_l2(out[f16][1], g_ref) < 1e-4
    # the 22-bit pairs are at least as close to the checker as the 16-bit ones (small-problem noise margin)
    assert rel_l2(out[1][0], hv_ref) <= 2.0 * rel_l2(out[0][0], hv_ref) + 1e-7


def test_mlp_hvp_linear_symmetric(ctx, port, mlp_path):  # test_oracle.cpp:107-132
    from oracle.bindings import blobs_dataset
    sizes = [30, 24, 6]
    X, y = blobs_dataset(64, 30, 6, seed=2)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(7)
    u, v = port.rng_normal(71, len(w)), port.rng_normal(72, len(w))
    b = d.Batch(X, y, 6)
    hu, hv, hc = mlp.hvp(w, u, b), mlp.hvp(w, v, b), mlp.hvp(w, 0.7 * u - 1.3 * v, b)
    assert rel_l2(hc, 0.7 * hu - 1.3 * hv) < 1e-5
    assert abs(u @ hv - v @ hu) <= 1e-4 * max(1.0, abs(u @ hv))


def test_mlp_pure_and_zero_case(ctx, mlp_path):  # test_oracle.cpp:68-79 and :152-160
    from paper_2505_00982_b200.config import synthetic_dataset
    data = synthetic_dataset("two-gaussians", 40, 23)
    mlp = d.MlpOracle(ctx, [2, 8, 2], "relu", "softmax_ce")
    w = mlp.init_params(9)
    b = d.Batch(data.features, data.labels, 2)
    g1, g2 = mlp.grad(w, b), mlp.grad(w, b)
    assert (g1 == g2).all()  # repeated calls are bitwise identical
    v = np.linspace(-1.0, 1.0, w.size)
    assert (mlp.hvp(w, v, b) == mlp.hvp(w, v, b)).all()
    z = d.MlpOracle(ctx, [2, 4, 1], "tanh", "mse")
    bz = d.Batch(np.array([[1.0, 2.0], [-1.0, 0.5], [0.0, 3.0]]), np.zeros(3), 0)
    wz = np.zeros(z.dim())
    assert z.value(wz, bz) == 0.0 and np.abs(z.grad(wz, bz)).max() == 0.0


def test_mlp_argument_errors(ctx):
    with pytest.raises(d.ArgumentError):
        d.MlpOracle(ctx, [2, 2])
    mlp = d.MlpOracle(ctx, [3, 4, 2])
    with pytest.raises(d.ArgumentError):
        mlp.value(np.zeros(mlp.dim()), d.Batch(np.zeros((4, 3)), np.zeros(4), 5))  # n_classes != outputs
    with pytest.raises(d.DimensionError):
        mlp.grad(np.zeros(3), d.Batch(np.zeros((4, 3)), np.zeros(4), 2))


def test_gemm_backends_agree_on_hvp(ctx, port):
    from oracle.bindings import blobs_dataset
    sizes = [784, 256, 10]
    X, y = blobs_dataset(128, 784, 10, seed=1)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    v = port.rng_normal(9, len(w))
    b = d.Batch(X, y, 10)
    ctx.set_option("gemm", 1)
    try:
        h1 = mlp.hvp(w, v, b)
    finally:
        ctx.set_option("gemm", 0)
    ctx.set_option("mlp_small", 0)
    try:
        h0 = mlp.hvp(w, v, b)
    finally:
        ctx.set_option("mlp_small", 1)
    assert rel_l2(h0, h1) < 2e-5


def test_hvp_cta_modes_vs_checker(ctx, ref):
    """Wide layers (several 256-row pair tiles, stream-K segments, narrow output layer): the
    single-CTA and CTA-pair GEMM kernels both match the reference HVP/gradient (fp64, OpenMP)
    to rel-L2 1e-4 and each other to 2e-5."""
    from oracle.bindings import blobs_dataset
    sizes = [512, 1024, 1024, 10]
    B = 512
    X, y = blobs_dataset(B, sizes[0], 10, seed=4)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(2)
    v = ref.rng_normal(8, len(w))
    b = d.Batch(X, y, 10)
    hv_ref = ref.mlp_hvp(sizes, w, v, X, y, 10)
    g_ref = ref.mlp_grad(sizes, w, X, y, 10)
    out = {}
    for cta in (1, 2):
        ctx.set_option("gemm_cta", cta)
        try:
            out[cta] = (mlp.hvp(w, v, b), mlp.grad(w, b))
        finally:
            ctx.set_option("gemm_cta", 0)
        assert rel_l2(out[cta][0], hv_ref) < 1e-4
        assert rel_l2(out[cta][1], g_ref) < 1e-4
    assert rel_l2(out[1][0], out[2][0]) < 2e-5
    assert rel_l2(out[1][1], out[2][1]) < 2e-5


# ------------------------------------------------------------------------------------ Lanczos
def random_symmetric(port, n, seed):  # test_support.hpp:65-72
    a = port.rng_normal(seed, n * n).reshape(n, n)
    return 0.5 * (a + a.T)


def run_lanczos(ctx, op, n, m, seed, k=0, l=0):
    st = d.lanczos_distributed(ctx, m, op, n, seed)
    ese = d.extract_ese_distributed(ctx, st, min(k, st.iterations), min(l, st.iterations - min(k, st.iterations)))
    return st, ese


def test_lanczos_dense_matches_checker(ctx, port):
    H = random_symmetric(port, 50, 123)
    st, ese = run_lanczos(ctx, d.dense_operator(ctx, H), 50, 20, 9, k=3, l=2)
    ref = port.lanczos(dict(kind=0, n=50, mat=H), 20, 9, k=3, l=2)
    hn = np.max(np.abs(np.linalg.eigvalsh(H)))
    assert st.iterations == ref["iterations"] == 20 and not st.breakdown
    # B entries within 1e-5 of ||H|| (fp32 basis, fp64 reductions)
    assert np.max(np.abs(st.tridiag.diag - ref["diag"])) <= 1e-5 * hn
    assert np.max(np.abs(st.tridiag.offdiag - ref["off"])) <= 1e-5 * hn
    assert np.max(np.abs(ese.eigvals - ref["eigvals"])) <= 1e-5 * hn
    D = st.basis_shard[:, :20]
    assert np.max(np.abs(D.T @ D - np.eye(20))) <= 1e-5  # test_lanczos.cpp:47-61 (fp32: 1e-5)
    T = np.diag(st.tridiag.diag) + np.diag(st.tridiag.offdiag[:19], 1) + np.diag(st.tridiag.offdiag[:19], -1)
    assert np.linalg.norm(D.T @ H @ D - T) <= 1e-4 * hn
    V = ese.eigvecs_shard(50)
    Vr = ref["eigvecs"]
    assert np.max(np.abs(V - Vr)) <= 1e-4  # same sign convention (lanczos.cpp:82-94)


def test_lanczos_galerkin_and_orthonormality(ctx, port):  # test_lanczos.cpp:47-61
    """D^T D = I and D^T H D = B on a random symmetric operator (fp32 basis: 1e-6 -> 2e-6 and 1e-5 ||H||)."""
    H = random_symmetric(port, 50, 123)
    st = d.lanczos_distributed(ctx, 20, d.dense_operator(ctx, H), 50, 9)
    assert st.iterations == 20
    Dm = st.basis_shard[:, :20]
    assert np.abs(Dm.T @ Dm - np.eye(20)).max() <= 2e-6
    B = np.diag(st.tridiag.diag) + np.diag(st.tridiag.offdiag[:19], 1) + np.diag(st.tridiag.offdiag[:19], -1)
    assert np.linalg.norm(Dm.T @ H @ Dm - B) <= 1e-5 * np.abs(np.linalg.eigvalsh(H)).max()


def test_lanczos_seed_determinism_bitwise(ctx, port):  # test_lanczos.cpp:85-93
    H = random_symmetric(port, 30, 5)
    op = d.dense_operator(ctx, H)
    a = d.lanczos_distributed(ctx, 12, op, 30, 21)
    b = d.lanczos_distributed(ctx, 12, op, 30, 21)
    c = d.lanczos_distributed(ctx, 12, op, 30, 22)
    assert (a.basis_shard == b.basis_shard).all() and (a.tridiag.diag == b.tridiag.diag).all()
    assert (a.tridiag.offdiag == b.tridiag.offdiag).all()
    assert not (c.tridiag.diag == a.tridiag.diag).all()


def test_lanczos_identity_breakdown(ctx):  # test_lanczos.cpp:22-33
    st, ese = run_lanczos(ctx, d.dense_operator(ctx, np.eye(6)), 6, 4, 11, k=1)
    assert st.breakdown and st.iterations == 1 and st.tridiag.dim() == 1
    assert abs(st.tridiag.diag[0] - 1.0) < 1e-6 and abs(ese.eigvals[0] - 1.0) < 1e-6


def test_lanczos_rank2_breakdown_matches(ctx, port):  # test_dist_lanczos.cpp:193-203
    H = np.zeros((12, 12))
    H[0, 0], H[1, 1] = 3.0, 1.0
    st, _ = run_lanczos(ctx, d.dense_operator(ctx, H), 12, 6, 13, k=1)
    ref = port.lanczos(dict(kind=0, n=12, mat=H), 6, 13, k=1)
    assert st.breakdown and st.iterations == ref["iterations"] < 6


def test_lanczos_diagonal_spectrum_exact(ctx):  # test_lanczos.cpp:35-45
    st, ese = run_lanczos(ctx, d.diagonal_operator(ctx, np.arange(1.0, 7.0)), 6, 6, 5, k=6)
    assert st.iterations == 6
    assert np.max(np.abs(np.sort(ese.eigvals) - np.arange(1.0, 7.0))) <= 1e-5


def test_extract_known_diagonal_signs(ctx):  # test_lanczos.cpp:95-111
    st, ese = run_lanczos(ctx, d.dense_operator(ctx, np.diag([10.0, 5.0, 1.0, 0.1])), 4, 4, 2, k=1, l=1)
    assert abs(ese.eigvals[0] - 10.0) <= 1e-5 and abs(ese.eigvals[1] - 0.1) <= 1e-5
    V = ese.eigvecs_shard(4)
    assert V[0, 0] >= 1 - 1e-5 and V[3, 1] >= 1 - 1e-5


def test_lanczos_nonfinite_hvp_raises(ctx, port):  # dist_lanczos.cpp:80-82
    H = random_symmetric(port, 30, 5)
    calls = []

    def hvp(v):
        calls.append(1)
        out = H @ v
        if len(calls) == 4:
            out[7] = np.nan
        return out

    with pytest.raises(d.NumericError, match="non-finite"):
        d.lanczos_distributed(ctx, 10, d.host_operator(ctx, hvp, 30), 30, 3)


def test_lanczos_rejects_bad_m(ctx):
    op = d.diagonal_operator(ctx, np.arange(1.0, 5.0))
    with pytest.raises(d.ArgumentError):
        d.lanczos_distributed(ctx, 5, op, 4, 1)
    st = d.lanczos_distributed(ctx, 4, op, 4, 1)
    with pytest.raises(d.ArgumentError):
        d.extract_ese_distributed(ctx, st, 3, 2)


def test_lanczos_host_operator(ctx, port):
    H = random_symmetric(port, 40, 5)
    st, ese = run_lanczos(ctx, d.host_operator(ctx, lambda v: H @ v, 40), 40, 12, 21, k=2, l=1)
    ref = port.lanczos(dict(kind=0, n=40, mat=H), 12, 21, k=2, l=1)
    assert np.max(np.abs(ese.eigvals - ref["eigvals"])) <= 1e-5 * np.max(np.abs(ref["eigvals"]))


def test_lanczos_large_diagonal(ctx, port):
    """GS passes at scale (many CTAs, chunked rows): n = 2^18, m = 40, spectrum 1 + (i mod 1000)."""
    n, m = 1 << 18, 40
    spec = 1.0 + (np.arange(n) % 1000)
    spec[:3] = [5000.0, 3000.0, 2000.0]
    st, ese = run_lanczos(ctx, d.diagonal_operator(ctx, spec), n, m, 99, k=4, l=2)
    ref = port.lanczos(dict(kind=1, n=n, mat=spec), m, 99, k=4, l=2, want_basis=False)
    assert np.max(np.abs(ese.eigvals - ref["eigvals"]) / np.abs(ref["eigvals"])) <= 1e-4
    assert np.max(np.abs(st.tridiag.diag - ref["diag"]) / np.max(spec)) <= 1e-5
    V, Vr = ese.eigvecs_shard(n), ref["eigvecs"]
    # ||V V^T - Vr Vr^T||_F^2 (sign-invariant; exact also when the fp32 Ritz vectors are not unit to 1e-7)
    proj = np.sum((V.T @ V) ** 2) + np.sum((Vr.T @ Vr) ** 2) - 2 * np.sum((V.T @ Vr) ** 2)
    assert np.sqrt(max(proj, 0.0)) <= 1e-4


def test_refresh_mlp_c1_eigenvalues(ctx, port):
    """SURVEY §8d per-refresh parity on identical inputs: C1 model 784-256-10, B=128, m=40, k=10."""
    from oracle.bindings import blobs_dataset
    sizes = [784, 256, 10]
    X, y = blobs_dataset(128, 784, 10, seed=7)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
    st, ese = run_lanczos(ctx, op, mlp.dim(), 40, 4242, k=10)
    ref = port.lanczos(dict(kind=2, n=mlp.dim(), sizes=sizes, w=w, X=X, y=y, ncls=10), 40, 4242, k=10,
                       want_basis=False)
    rel = np.abs(ese.eigvals - ref["eigvals"]) / np.abs(ref["eigvals"])
    assert rel.max() <= 1e-4, rel  # north-star bound: eigenvalues within 1e-4 relative
    assert st.iterations == ref["iterations"]


# ------------------------------------------------------------------------------------ update
@pytest.mark.parametrize("fused", [1, 0], ids=["one-launch", "three-pass"])
@pytest.mark.parametrize("kind", ["sgd", "momentum", "adam", "adamw"])
@pytest.mark.parametrize("admm", [False, True])
def test_deltas_vs_checker(ctx, port, kind, admm, fused):
    """The update passes (fused into one cooperative launch at small n, option upd_small; or the three
    bandwidth passes) against the checker's BaseOptimizer / split_deltas sequence."""
    from oracle.bindings import base_cfg
    ctx.set_option("upd_small", fused)
    n, r, T = 20000, 8, 4
    V = np.linalg.qr(port.rng_normal(1, n * r).reshape(n, r))[0]
    ev = np.array([50.0, 20.0, 7.0, 3.0, 1e-9, -1e-13, -2.0, 0.5])
    g = port.rng_normal(2, T * n).reshape(T, n)
    pi = port.rng_normal(3, n) if admm else None
    w = port.rng_normal(4, n)
    sigma = 0.05 if admm else 0.0
    cfg = d.BaseConfig(kind, lr=1e-2)
    opt = d.BaseOptimizer(ctx, cfg, n)
    ese = d.EseResult.from_host(ctx, ev, V)
    nw_ref, bs_ref, _ = port.deltas_seq(base_cfg(kind, lr=1e-2), ev, V, g, w, 0.3, pi=pi, sigma=sigma)
    for t in range(T):
        dl = d.admm_deltas(g[t], pi, ese, opt, w, 0.3, sigma) if admm else d.fosi_deltas(g[t], ese, opt, w, 0.3)
        # update pass fed identical g, pi, w, V: per-element within 2e-6 of the vector's max (fp32)
        assert np.max(np.abs(dl.newton - nw_ref[t])) <= 2e-6 * np.max(np.abs(nw_ref[t]))
        assert np.max(np.abs(dl.base - bs_ref[t])) <= 5e-6 * np.max(np.abs(bs_ref[t]))
    ctx.set_option("upd_small", 1)


@pytest.mark.parametrize("n,r", [(4099, 33), (65537, 48), (3001, 50), (512, 1)])
@pytest.mark.parametrize("kind", ["momentum", "adamw"])
def test_deltas_shapes(ctx, port, n, r, kind):
    """Update passes across subspace ranks (bulk-copy staged P2 for r <= 48, register-staged above)
    and partial final chunks."""
    from oracle.bindings import base_cfg
    T = 2
    V = np.linalg.qr(port.rng_normal(11, n * r).reshape(n, r))[0]
    ev = np.linspace(40.0, -3.0, r)
    g = port.rng_normal(12, T * n).reshape(T, n)
    pi = port.rng_normal(13, n)
    w = port.rng_normal(14, n)
    cfg = d.BaseConfig(kind, lr=1e-2)
    opt = d.BaseOptimizer(ctx, cfg, n)
    ese = d.EseResult.from_host(ctx, ev, V)
    nw_ref, bs_ref, _ = port.deltas_seq(base_cfg(kind, lr=1e-2), ev, V, g, w, 0.3, pi=pi, sigma=0.05)
    den = np.maximum(np.abs(ev), 1e-6) + 0.05
    for t in range(T):
        dl = d.admm_deltas(g[t], pi, ese, opt, w, 0.3, 0.05)
        # fp32 dots: error relative to the magnitudes summed, alpha |V| (|V|^T |g + pi| / den), not to the
        # (possibly cancelled) result
        scale_n = max(np.max(np.abs(nw_ref[t])), 0.3 * np.max(np.abs(V) @ ((np.abs(V).T @ np.abs(g[t] + pi)) / den)))
        assert np.max(np.abs(dl.newton - nw_ref[t])) <= 2e-6 * scale_n
        if kind == "adamw":
            # Adam's first steps are sign-like (m/sqrt(v) = g/|g|): an element whose g2 = g - V c sits at
            # fp32 rounding level can flip, so the base part is compared in norm
            assert rel_l2(dl.base, bs_ref[t]) <= 1e-5
        else:
            assert np.max(np.abs(dl.base - bs_ref[t])) <= 5e-6 * np.max(np.abs(bs_ref[t]))


def test_deltas_known_answers(ctx):  # test_optimizer.cpp:78-199
    V = np.array([[1.0], [0.0]])
    ese = d.EseResult.from_host(ctx, [4.0], V)
    zero = d.BaseOptimizer(ctx, d.BaseConfig("sgd", lr=0.0), 2)
    dl = d.fosi_deltas([4.0, 1.0], ese, zero, [0.0, 0.0], 1.0)
    assert abs(dl.newton[0] + 1.0) < 1e-6 and dl.newton[1] == 0.0 and np.abs(dl.base).max() == 0.0
    dl = d.admm_deltas([4.0, 1.0], [0.0, 0.0], ese, zero, [0.0, 0.0], 1.0, 1.0)
    assert abs(dl.newton[0] + 0.8) < 1e-6
    adam = d.BaseOptimizer(ctx, d.BaseConfig("adam", lr=1e-3), 3)
    g = np.array([0.5, -2.0, 3.0])
    assert np.allclose(adam.step(g, np.zeros(3)), -1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-6)
    with pytest.raises(d.NumericError):
        d.BaseOptimizer(ctx, d.BaseConfig("adam"), 2).step([1.0, np.inf], [0.0, 0.0])


def test_delta_orthogonality_random_draws(ctx, port):  # test_optimizer.cpp:201-227
    """Newton and base deltas are orthogonal (base lives in the complement of span(V_hat)) over 25 draws;
    fp32 device arithmetic: |<newton, base>| <= 1e-6 |newton| |base| (reference: 1e-8 in fp64)."""
    H = random_symmetric(port, 12, 7)
    w, U = np.linalg.eigh(H)
    idx = list(np.argsort(-w)[:3]) + [int(np.argmin(w))]
    ese = d.EseResult.from_host(ctx, w[idx], U[:, idx])
    opt = d.BaseOptimizer(ctx, d.BaseConfig("adam"), 12)
    draws = port.rng_normal(4242, 25 * 24).reshape(25, 24)
    for t in range(25):
        g, pi = draws[t, :12], draws[t, 12:]
        dl = d.admm_deltas(g, pi, ese, opt, np.zeros(12), 0.2, 0.05)
        dot = float(np.dot(dl.newton, dl.base))
        assert abs(dot) <= max(1e-6 * np.linalg.norm(dl.newton) * np.linalg.norm(dl.base), 1e-12)


def test_optimizer_reference_cases(ctx, port):  # test_optimizer.cpp:55-71, :171-186, :229-244
    mom = d.BaseOptimizer(ctx, d.BaseConfig("momentum", lr=0.5), 2)
    assert np.abs(mom.step([0.0, 0.0], [1.0, 1.0])).max() == 0.0  # zero gradient, zero moments
    adamw = d.BaseOptimizer(ctx, d.BaseConfig("adamw", lr=0.1, weight_decay=0.05), 2)
    dw = adamw.step([0.0, 0.0], [2.0, -4.0])  # pure decoupled decay
    assert np.allclose(dw, [-0.1 * 0.05 * 2.0, 0.1 * 0.05 * 4.0], rtol=1e-6, atol=0)
    # admm_deltas(pi = 0, sigma = 0) == fosi_deltas
    H = random_symmetric(port, 8, 99)
    w_, U = np.linalg.eigh(H)
    idx = [int(np.argmax(w_)), int(np.argsort(-w_)[1]), int(np.argmin(w_))]
    ese = d.EseResult.from_host(ctx, w_[idx], U[:, idx])
    g, w = port.rng_normal(98, 8), port.rng_normal(97, 8)
    a, b = d.BaseOptimizer(ctx, d.BaseConfig("adam"), 8), d.BaseOptimizer(ctx, d.BaseConfig("adam"), 8)
    f = d.fosi_deltas(g, ese, a, w, 0.3)
    m = d.admm_deltas(g, np.zeros(8), ese, b, w, 0.3, 0.0)
    assert np.abs(f.newton - m.newton).max() <= 1e-7 * np.abs(f.newton).max()
    assert np.abs(f.base - m.base).max() <= 1e-7 * np.abs(f.base).max()
    # the eigenvalue floor keeps the Newton step finite and the negative direction's sign
    V = np.zeros((3, 2))
    V[0, 0] = V[1, 1] = 1.0
    ese = d.EseResult.from_host(ctx, [1e-12, -1e-13], V)
    zero = d.BaseOptimizer(ctx, d.BaseConfig("sgd", lr=0.0), 3)
    dl = d.fosi_deltas([1.0, 1.0, 1.0], ese, zero, np.zeros(3), 1.0, 1e-6)
    assert np.isfinite(dl.newton).all() and abs(dl.newton[0]) <= 1.0 / 1e-6 + 1.0 and dl.newton[1] > 0.0


def test_admm_round(ctx, port):
    n = 1000
    w_a, pi, w_a2 = port.rng_normal(1, n), port.rng_normal(2, n), port.rng_normal(3, n)
    st = d.make_admm_state(w_a, 0.7)
    st.pi = pi
    d.admm_w_update(ctx, st)
    w_ref, pi_ref = port.admm_round(0.7, w_a, pi, w_a2)
    assert np.max(np.abs(st.w - w_ref)) <= 1e-6 * np.max(np.abs(w_ref))
    st.w_a = w_a2
    d.admm_dual_update(ctx, st)
    assert np.max(np.abs(st.pi - pi_ref)) <= 1e-5 * np.max(np.abs(pi_ref))
    with pytest.raises(d.ArgumentError):
        d.make_admm_state(w_a, 0.0)


@pytest.mark.parametrize("n,m,k,l", [(50_000, 80, 32, 0), (70_001, 40, 10, 3), (9_000, 96, 50, 14), (4_096, 20, 1, 0),
                                     (30_000, 100, 20, 0)])
def test_ritz_tensor_core_matches_cuda_core(ctx, port, n, m, k, l):
    """Ritz vectors V = D U' on the tensor cores (tcgen05 kind::tf32, 3xTF32 split, ~2^-21 of sum |D||U'|)
    agree with the fp32 CUDA-core kernel: entries within 1e-5 of max|V| (the Ritz combinations cancel,
    so entry-relative bounds are meaningless) and projectors within 3e-5 (SURVEY §8d bar: 1e-4; the
    split's error grows with the K = m + 1 of the sums: 1.3e-5 measured at m = 100)."""
    spec = 1.0 + (np.arange(n) % 997) * 0.37 + 0.01 * port.rng_normal(3, n)
    op = d.diagonal_operator(ctx, spec)
    st = d.lanczos_distributed(ctx, m, op, n, 17)
    ke = min(k, st.iterations)
    le = min(l, st.iterations - ke)
    out = []
    for tc in (0, 1):
        ctx.set_option("ritz_tc", tc)
        try:
            ese = d.extract_ese_distributed(ctx, st, ke, le)
            out.append((ese.eigvals, ese.eigvecs_shard(n)))
        finally:
            ctx.set_option("ritz_tc", 1)
    assert (out[0][0] == out[1][0]).all()
    V0, V1 = out[0][1], out[1][1]
    assert np.max(np.abs(V1 - V0)) <= 1e-5 * np.max(np.abs(V0))
    G = V0.T @ V1  # ||V1 V1^T - V0 V0^T||_F^2 = tr(V0^T V0)^2-ish terms, evaluated without n x n matrices
    proj2 = np.sum((V0.T @ V0) ** 2) + np.sum((V1.T @ V1) ** 2) - 2 * np.sum(G ** 2)
    assert np.sqrt(max(proj2, 0.0)) <= 3e-5


@pytest.mark.parametrize("n,m,k,l", [(20_000, 80, 32, 0), (9_000, 40, 10, 3), (4_096, 2, 1, 1), (60_000, 512, 128, 0),
                                     (30_000, 900, 16, 16), (3_000, 1, 1, 0)])
def test_tql2_split_matches_single_cta(ctx, n, m, k, l):
    """The split eigensolve (QL chain producing a rotation log, consumer CTAs replaying it concurrently
    from shared memory, then selection) replays the single-CTA tql2's rotations in the same order with
    the same arithmetic: eigenvalues and Ritz vectors bit-identical, at m = 1 (no sweep), small m, the C4 m = 80, the C5 m = 512 and m = 900 (16-column
    replay CTAs)."""
    spec = 1.0 + np.sin(np.arange(n) * 0.731) * 3.0 + (np.arange(n) % 7 == 0) * 0.5
    op = d.diagonal_operator(ctx, spec)
    st = d.lanczos_distributed(ctx, m, op, n, 5)
    ke = min(k, st.iterations)
    le = min(l, st.iterations - ke)
    out = []
    for split in (0, 1):
        ctx.set_option("tql2_split", split)
        try:
            ese = d.extract_ese_distributed(ctx, st, ke, le)
            out.append((ese.eigvals, ese.eigvecs_shard(n)))
        finally:
            ctx.set_option("tql2_split", 1)
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


def test_tql2_log_overflow_falls_back_bit_identical(ctx):
    """The split eigensolve's rotation log is sized for typical QL (2 m^2 entries, not the reference's
    worst case of 30 m (m - 1)); a log that fills up stops the kernel with status 2 and the single-CTA
    eigensolve redoes the extraction: results bit-identical to the unconstrained split form."""
    n, m = 20_000, 80
    spec = 1.0 + np.sin(np.arange(n) * 0.731) * 3.0
    st = d.lanczos_distributed(ctx, m, d.diagonal_operator(ctx, spec), n, 5)
    ref = d.extract_ese_distributed(ctx, st, 8, 2)
    e0, v0 = ref.eigvals, ref.eigvecs_shard(n)
    before = ctx.stat("tql2_log_overflows")
    ctx.set_option("tql2_log_cap", 200)
    try:
        ese = d.extract_ese_distributed(ctx, st, 8, 2)
    finally:
        ctx.set_option("tql2_log_cap", 0)
    assert ctx.stat("tql2_log_overflows") == before + 1
    assert np.array_equal(ese.eigvals, e0) and np.array_equal(ese.eigvecs_shard(n), v0)


def test_nccl_collectives_one_rank(ctx):
    """The NCCL path of every collective wrapper (run-time libnccl binding, 1-rank communicator,
    datatypes, counts, stream order) and the ledger rows it records."""
    import ctypes as C
    from paper_2505_00982_b200._lib import lib
    ctx.reset_accounting()
    err = C.c_double(-1.0)
    d.check(lib.dho2g_test_collectives(ctx.h, C.byref(err)))
    assert err.value == 0.0
    rows = ctx.ledger()
    assert [r[1] for r in rows] == ["all_gather", "reduce_scatter", "all_reduce", "all_reduce"]
    assert all(r[4] == 0 and r[5] == 0 for r in rows)  # one rank: no traffic
    ctx.reset_accounting()


def test_nccl_collectives_captured_in_graph(ctx):
    """The multi-rank refresh graph captures its NCCL calls: all-gather, reduce-scatter and the ordered
    fp64 all-reduce captured into a CUDA graph on a 1-rank NCCL communicator, replayed twice, exact."""
    import ctypes as C
    from paper_2505_00982_b200._lib import lib
    err = C.c_double(-1.0)
    d.check(lib.dho2g_test_collectives_graph(ctx.h, C.byref(err)))
    assert err.value == 0.0


def test_missing_rank_is_deadlock_error():
    """test_collectives.cpp:245-258 on the device path: a rank that never joins surfaces as
    DeadlockError after the timeout (non-blocking NCCL init + polling + abort), not a hang. Run in a
    child process so a misbehaving NCCL teardown cannot take the test session with it."""
    import subprocess
    import sys
    code = (
        "import time, paper_2505_00982_b200 as d\n"
        "c = d.Context(0)\n"
        "c.set_option('nccl_timeout_s', 3)\n"
        "t0 = time.time()\n"
        "try:\n"
        "    c.comm_init(d.Context.nccl_unique_id(), 0, 2)\n"
        "    print('NO ERROR')\n"
        "except d.DeadlockError as e:\n"
        "    print('DEADLOCK', round(time.time() - t0, 1), c.world, e)\n"
        "try:\n"  # the failed context refuses further work instead of running on as one rank
        "    d.MlpOracle(c, [2, 3, 2])\n"
        "    print('STILL USABLE')\n"
        "except d.NcclError as e:\n"
        "    print('FAILED CONTEXT', e)\n"
    )
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=180)
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("DEADLOCK")]
    assert line, out.stdout + out.stderr
    secs, world = line[0].split()[1:3]
    assert 2.5 <= float(secs) < 60 and world == "2"
    assert "timed out on rank 0" in out.stdout
    assert "FAILED CONTEXT" in out.stdout and "unusable after a failed collective" in out.stdout
