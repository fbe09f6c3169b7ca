"""Pins the fp64 torch mirror (tests/fp64_mirror.py, test infrastructure for the parity-at-scale tests) to
the CPU checkers on the CPU: the compiled reference where /root/reference was available at build time,
the pinned C restatement otherwise. Bounds are fp64-vs-fp64 (summation order only)."""
import numpy as np
import pytest
import torch

import fp64_mirror as M
from oracle.bindings import base_cfg, blobs_dataset

CPU = torch.device("cpu")


@pytest.fixture(scope="module")
def chk():
    from oracle.bindings import CpuChecker, reference_available
    return CpuChecker("reference" if reference_available() else "port")


def T(a):
    return torch.tensor(np.asarray(a, np.float64), dtype=torch.float64)


@pytest.mark.parametrize("sizes,act,loss,ncls", [([20, 16, 12, 5], "tanh", "softmax_ce", 5),
                                                 ([20, 16, 12, 5], "relu", "softmax_ce", 5),
                                                 ([13, 24, 1], "tanh", "mse", 0),
                                                 ([30, 24, 24, 6], "tanh", "mse", 6)])
def test_mirror_mlp_matches_reference(chk, sizes, act, loss, ncls):
    X, y = blobs_dataset(37, sizes[0], max(ncls, 1), seed=11)
    if ncls == 0:
        y = np.sin(np.arange(37) * 0.37)
    w = chk.mlp_init(sizes, 3) + 0.05 * chk.rng_normal(5, chk.mlp_dim(sizes))
    v = chk.rng_normal(6, len(w))
    a, lo = {"tanh": 0, "relu": 1}[act], {"softmax_ce": 0, "mse": 1}[loss]
    mir = M.MlpMirror(sizes, CPU, act, loss)
    assert mir.n == len(w)
    hv = mir.hvp(T(w), T(v), T(X), T(y)).numpy()
    g = mir.grad(T(w), T(X), T(y)).numpy()
    hv_r = chk.mlp_hvp(sizes, w, v, X, y, ncls, a, lo)
    g_r = chk.mlp_grad(sizes, w, X, y, ncls, a, lo)
    assert np.max(np.abs(hv - hv_r)) <= 1e-12 * np.max(np.abs(hv_r))
    assert np.max(np.abs(g - g_r)) <= 1e-12 * np.max(np.abs(g_r))
    assert abs(mir.value(T(w), T(X), T(y)) - chk.mlp_value(sizes, w, X, y, ncls, a, lo)) <= 1e-12
    if ncls:
        assert mir.accuracy(T(w), T(X), T(y)) == chk.mlp_accuracy(sizes, w, X, y, ncls, a, lo)


def test_mirror_lanczos_and_extract_match_reference(chk):
    sizes = [30, 24, 24, 6]
    X, y = blobs_dataset(64, 30, 6, seed=2)
    w = chk.mlp_init(sizes, 7)
    n = len(w)
    mir = M.MlpMirror(sizes, CPU)
    mir.prepare(T(w), T(X), T(y))
    lz = M.lanczos(chk, mir.hvp_prepared, n, 24, 77, CPU)
    ev, V = M.extract_ese(chk, lz, 5, 2)
    ref = chk.lanczos(dict(kind=2, n=n, sizes=sizes, w=w, X=X, y=y, ncls=6), 24, 77, k=5, l=2)
    hn = np.abs(ref["eigvals"]).max()
    assert lz["iterations"] == ref["iterations"] and lz["breakdown"] == ref["breakdown"]
    assert np.max(np.abs(lz["diag"] - ref["diag"])) <= 1e-10 * hn
    assert np.max(np.abs(lz["off"] - ref["off"][: len(lz["off"])])) <= 1e-10 * hn
    assert np.max(np.abs(ev - ref["eigvals"])) <= 1e-10 * hn
    assert np.max(np.abs(V.numpy().T - ref["eigvecs"])) <= 1e-8  # same sign convention


def test_mirror_lanczos_breakdown_matches_reference(chk):
    H = np.zeros((12, 12))
    H[0, 0], H[1, 1] = 3.0, 1.0
    Ht = T(H)
    lz = M.lanczos(chk, lambda v: Ht @ v, 12, 6, 13, CPU)
    ref = chk.lanczos(dict(kind=0, n=12, mat=H), 6, 13, k=1)
    assert lz["breakdown"] and lz["iterations"] == ref["iterations"]


@pytest.mark.parametrize("kind", ["momentum", "adamw"])
def test_mirror_split_deltas_match_reference(chk, kind):
    n, r, Tn = 3000, 6, 3
    V = np.linalg.qr(chk.rng_normal(1, n * r).reshape(n, r))[0]
    ev = np.array([50.0, 7.0, 1e-9, 0.0, -0.01, -2.0])  # floor, zero and the |den| < floor branch (sigma 0.01)
    g = chk.rng_normal(2, Tn * n).reshape(Tn, n)
    pi, w = chk.rng_normal(3, n), chk.rng_normal(4, n)
    nw_r, bs_r, w_r = chk.deltas_seq(base_cfg(kind, lr=1e-2), ev, V, g, w, 0.3, pi=pi, sigma=0.01, advance=True)
    opt = M.BaseOptimizerMirror(kind, n, CPU, lr=1e-2)
    wt, Vt = T(w), T(V.T)
    for t in range(Tn):
        nw, bs, *_ = M.split_deltas(T(g[t]), T(pi), ev, Vt, opt, wt, 0.3, 0.01, 1e-6)
        assert np.max(np.abs(nw.numpy() - nw_r[t])) <= 1e-12 * np.max(np.abs(nw_r[t]))
        assert np.max(np.abs(bs.numpy() - bs_r[t])) <= 1e-10 * np.max(np.abs(bs_r[t]))
        wt = wt + bs + nw
    assert np.max(np.abs(wt.numpy() - w_r)) <= 1e-10 * np.max(np.abs(w_r))


def test_hashed_inputs_match_c_generator():
    """tests/scale_inputs.py's counter hash in numpy and torch gives the same bits (the C copy in
    oracle/ref_shim.cpp is pinned through the c4_update fixture's w_after at step 0 inputs)."""
    import scale_inputs as S
    idx = np.array([0, 1, 2, 12345, (1 << 24) - 1, 1 << 24, 100_989_961, 123_456_789], np.int64)
    for salt in (2, 3, 10, 131):
        a = S.unif_np(idx, salt, 2.0 ** -6)
        b = S.unif_torch(torch.tensor(idx), salt, 2.0 ** -6, torch.float64).numpy()
        assert (a == b).all()
        assert (a.astype(np.float32).astype(np.float64) == a).all()  # fp32-exact
    big = S.unif_np(np.arange(1 << 20, dtype=np.int64), 5, 1.0)
    assert abs(big.mean()) < 3e-3 and abs(big.std() - 1 / np.sqrt(3)) < 3e-3  # ~U(-1, 1)
