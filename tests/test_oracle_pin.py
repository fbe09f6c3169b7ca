"""Pins the CPU checker (oracle/dho2_oracle.c) before anything is compared against it.

1. Bitwise against the UNMODIFIED reference library (oracle/_ref/libdho2ref.so) on the same inputs.
2. Against the known-answer cases of the reference's own doctest suites, with
   numpy fp64 standing in for Eigen (test_support.hpp:90-93).
3. Against the committed golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py
   from the reference library), so the pin holds where the reference is not present.
"""
import os

import numpy as np
import pytest

from oracle.bindings import base_cfg, blobs_dataset, train_cfg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def small_mlp(port, sizes=(20, 16, 12, 5), B=37, seed=3):
    X, y = blobs_dataset(B, sizes[0], sizes[-1], seed=seed)
    w = port.mlp_init(list(sizes), 1)
    w = w + 0.01 * port.rng_normal(4, len(w))
    return list(sizes), X, y, w


# ------------------------------------------------------------------------------------ bitwise
def test_rng_streams_bitwise(port, ref):
    for seed in (0, 1, 5, 2**63 + 11):
        assert (port.rng_u64(seed, 257) == ref.rng_u64(seed, 257)).all()
        assert (port.rng_normal(seed, 101) == ref.rng_normal(seed, 101)).all()
        assert (port.rng_uniform(seed, 33) == ref.rng_uniform(seed, 33)).all()
        assert (port.shuffle_iota(seed, 1000) == ref.shuffle_iota(seed, 1000)).all()


def test_bookkeeping_bitwise(port, ref):
    for n, C in [(10, 8), (203530, 4), (12, 5), (1, 3), (100989962, 8)]:
        for r in range(C):
            assert port.shard(n, C, r) == ref.shard(n, C, r)
    for k, l, n in [(8, 0, 10000), (1, 1, 100), (3, 2, 10), (10, 0, 203530), (20, 0, 10510346), (32, 0, 100989962)]:
        assert port.lanczos_budget(k, l, n) == ref.lanczos_budget(k, l, n)
    assert (port.epoch_permutation(1280, 7, 3) == ref.epoch_permutation(1280, 7, 3)).all()
    assert (port.seeded_unit_gaussian(777, 9) == ref.seeded_unit_gaussian(777, 9)).all()


@pytest.mark.parametrize("act", [0, 1])
@pytest.mark.parametrize("loss", [0, 1])
def test_mlp_bitwise(port, ref, act, loss):
    sizes, X, y, w = small_mlp(port)
    v = port.rng_normal(8, len(w))
    assert (port.mlp_init(sizes, 1) == ref.mlp_init(sizes, 1)).all()
    assert (port.mlp_hvp(sizes, w, v, X, y, 5, act, loss) == ref.mlp_hvp(sizes, w, v, X, y, 5, act, loss)).all()
    assert (port.mlp_grad(sizes, w, X, y, 5, act, loss) == ref.mlp_grad(sizes, w, X, y, 5, act, loss)).all()
    assert port.mlp_value(sizes, w, X, y, 5, act, loss) == ref.mlp_value(sizes, w, X, y, 5, act, loss)
    assert port.mlp_accuracy(sizes, w, X, y, 5, act, loss) == ref.mlp_accuracy(sizes, w, X, y, 5, act, loss)


def test_tridiag_bitwise(port, ref):
    d, e = port.rng_normal(3, 40), port.rng_normal(4, 39)
    a, A = port.tridiag_eig(d, e)
    b, Bv = ref.tridiag_eig(d, e)
    assert (a == b).all() and (A == Bv).all()


@pytest.mark.parametrize("workers", [1, 2, 3, 5])
def test_lanczos_mlp_bitwise(port, ref, workers):
    sizes, X, y, w = small_mlp(port)
    op = dict(kind=2, n=len(w), sizes=sizes, w=w, X=X, y=y, ncls=5)
    a = port.lanczos(op, 20, 77, k=4, l=2, workers=workers)
    b = ref.lanczos(op, 20, 77, k=4, l=2, workers=workers)
    for key in ("diag", "off", "basis", "eigvals", "eigvecs"):
        assert (a[key] == b[key]).all(), key
    assert a["iterations"] == b["iterations"] and a["safeguard_passes"] == b["safeguard_passes"]


def test_lanczos_breakdown_bitwise(port, ref):
    H = np.zeros((12, 12))
    H[0, 0], H[1, 1] = 3.0, 1.0
    a = port.lanczos(dict(kind=0, n=12, mat=H), 6, 13, k=1, workers=3)
    b = ref.lanczos(dict(kind=0, n=12, mat=H), 6, 13, k=1, workers=3)
    assert a["breakdown"] and b["breakdown"] and a["iterations"] == b["iterations"] < 6
    assert (a["diag"] == b["diag"]).all() and (a["off"] == b["off"]).all() and (a["eigvals"] == b["eigvals"]).all()


@pytest.mark.parametrize("kind", ["sgd", "momentum", "adam", "adamw"])
def test_deltas_bitwise(port, ref, kind):
    n, r = 50, 3
    V = np.linalg.qr(port.rng_normal(1, n * r).reshape(n, r))[0]
    ev = np.array([5.0, 1e-9, -2.0])
    g = port.rng_normal(2, 4 * n).reshape(4, n)
    pi = port.rng_normal(3, n)
    w = port.rng_normal(4, n)
    c = base_cfg(kind, lr=1e-2)
    for p in (None, pi):
        a = port.deltas_seq(c, ev, V, g, w, 0.3, pi=p, sigma=0.05 if p is not None else 0.0, advance=True)
        b = ref.deltas_seq(c, ev, V, g, w, 0.3, pi=p, sigma=0.05 if p is not None else 0.0, advance=True)
        for x, y_ in zip(a, b):
            assert (x == y_).all()


@pytest.mark.parametrize("trainer,base,workers", [("dho2", "adam", 1), ("dho2", "momentum", 3), ("fosi", "adamw", 2),
                                                  ("sgd", "sgd", 2)])
def test_train_bitwise(port, ref, trainer, base, workers):
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(200, 20, 5, seed=7)
    w0 = port.mlp_init(sizes, 2)
    cfg = train_cfg(trainer, base_cfg(base), k=3, l=1, outer_rounds=2, inner_epochs=2, epochs=3, batch_size=16,
                    curvature_batch=40, seed=21)
    a = port.train_mlp(cfg, sizes, X, y, w0, workers=workers, ncls=5)
    b = ref.train_mlp(cfg, sizes, X, y, w0, workers=workers, ncls=5)
    assert (a["w_final"] == b["w_final"]).all()
    assert (a["loss"] == b["loss"]).all() and a["refreshes"] == b["refreshes"]
    np.testing.assert_array_equal(a["resid"], b["resid"])


# ------------------------------------------------------------------------------------ known answers
def test_budget_known_answers(port):  # test_lanczos.cpp:12-20
    assert port.lanczos_budget(8, 0, 10000) == 32
    assert port.lanczos_budget(1, 1, 100) == 10
    assert port.lanczos_budget(3, 2, 10) == 10
    from oracle.bindings import CheckerError
    for k, l in [(6, 5), (0, 0)]:
        with pytest.raises(CheckerError):
            port.lanczos_budget(k, l, 10)


def test_shard_known_answer(port):  # n=10, C=8 -> 2,2,2,2,2,0,0,0
    assert [port.shard(10, 8, r)[1] - port.shard(10, 8, r)[0] for r in range(8)] == [2, 2, 2, 2, 2, 0, 0, 0]


def test_tridiag_known_answers(port):  # test_linalg.cpp:38-99
    vals, _ = port.tridiag_eig([2, 2], [1])
    assert abs(vals[0] - 1) < 1e-12 and abs(vals[1] - 3) < 1e-12
    vals, U = port.tridiag_eig(np.ones(5), np.zeros(4))
    assert np.allclose(vals, 1, atol=1e-14)
    d, e = port.rng_normal(33, 12), port.rng_normal(34, 11)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    vals, U = port.tridiag_eig(d, e)
    assert np.max(np.abs(vals - np.linalg.eigvalsh(T))) <= 1e-9
    assert np.linalg.norm(U @ np.diag(vals) @ U.T - T) <= 1e-8
    assert np.linalg.norm(U.T @ U - np.eye(12)) <= 1e-10


def test_lanczos_known_answers(port):  # test_lanczos.cpp:22-111
    a = port.lanczos(dict(kind=0, n=6, mat=np.eye(6)), 4, 11, k=1)
    assert a["breakdown"] and a["iterations"] == 1 and abs(a["diag"][0] - 1) < 1e-14
    a = port.lanczos(dict(kind=0, n=6, mat=np.diag(np.arange(1.0, 7.0))), 6, 5, k=0)
    vals, _ = port.tridiag_eig(a["diag"], a["off"][:5])
    assert np.max(np.abs(vals - np.arange(1.0, 7.0))) <= 1e-8
    a = port.lanczos(dict(kind=0, n=4, mat=np.diag([10.0, 5.0, 1.0, 0.1])), 4, 2, k=1, l=1)
    assert abs(a["eigvals"][0] - 10) <= 1e-7 and abs(a["eigvals"][1] - 0.1) <= 1e-7
    V = a["eigvecs"]
    assert V[0, 0] >= 1 - 1e-6 and V[3, 1] >= 1 - 1e-6


def test_optimizer_known_answers(port):  # test_optimizer.cpp:31-199
    d = port.base_steps(base_cfg("adam", lr=1e-3), np.array([[0.5, -2.0, 3.0]]), np.zeros(3))[0]
    g = np.array([0.5, -2.0, 3.0])
    assert np.allclose(d, -1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-12)
    d = port.base_steps(base_cfg("adamw", lr=0.1, weight_decay=0.05), np.zeros((1, 2)), np.array([2.0, -4.0]))[0]
    assert np.allclose(d, [-0.1 * 0.05 * 2.0, 0.1 * 0.05 * 4.0], rtol=1e-12)
    V = np.array([[1.0], [0.0]])
    nw, bs, _ = port.deltas_seq(base_cfg("sgd", lr=0.0), [4.0], V, np.array([[4.0, 1.0]]), np.zeros(2), 1.0)
    assert abs(nw[0, 0] + 1.0) < 1e-14 and nw[0, 1] == 0.0 and np.abs(bs).max() == 0.0
    nw, bs, _ = port.deltas_seq(base_cfg("sgd", lr=0.0), [4.0], V, np.array([[4.0, 1.0]]), np.zeros(2), 1.0,
                                pi=np.zeros(2), sigma=1.0)
    assert abs(nw[0, 0] + 4.0 / 5.0) < 1e-14


# ------------------------------------------------------------------------------------ golden fixtures
def test_golden_fixtures(port):
    path = os.path.join(GOLDEN, "golden.npz")
    if not os.path.exists(path):
        pytest.skip("golden fixtures not generated")
    G = np.load(path)
    sizes = list(G["mlp_sizes"])
    assert (port.mlp_hvp(sizes, G["mlp_w"], G["mlp_v"], G["mlp_X"], G["mlp_y"], 5) == G["mlp_hv"]).all()
    assert (port.mlp_grad(sizes, G["mlp_w"], G["mlp_X"], G["mlp_y"], 5) == G["mlp_g"]).all()
    op = dict(kind=2, n=len(G["mlp_w"]), sizes=sizes, w=G["mlp_w"], X=G["mlp_X"], y=G["mlp_y"], ncls=5)
    a = port.lanczos(op, int(G["lz_m"]), int(G["lz_seed"]), k=4, l=2, workers=3)
    assert (a["diag"] == G["lz_diag"]).all() and (a["eigvals"] == G["lz_eigvals"]).all()
    cfg = train_cfg("dho2", base_cfg("momentum"), k=3, l=1, outer_rounds=2, inner_epochs=2, batch_size=16,
                    curvature_batch=40, seed=21)
    t = port.train_mlp(cfg, sizes, G["tr_X"], G["tr_y"], G["tr_w0"], workers=2, ncls=5)
    assert (t["w_final"] == G["tr_wfinal"]).all() and (t["loss"] == G["tr_loss"]).all()


# ------------------------------------------------------------------------------------ QuadraticOracle
# oracle.cpp:233-286: rotation, apply_h / value, Lanczos and train() on it.
@pytest.mark.parametrize("n,seed", [(1, 5), (6, 3), (40, 9), (60, 4)])
def test_quadratic_bitwise(port, ref, n, seed):
    assert (port.quadratic_rotation(n, seed) == ref.quadratic_rotation(n, seed)).all()
    spec = 0.5 + np.arange(float(n))
    x = port.rng_normal(seed + 1, n)
    for rs in (0, seed):
        a, va = port.quadratic_apply(spec, rs, x)
        b, vb = ref.quadratic_apply(spec, rs, x)
        assert (a == b).all() and va == vb


@pytest.mark.parametrize("workers", [1, 3])
def test_lanczos_rotated_quadratic_bitwise(port, ref, workers):
    spec = np.random.default_rng(200).uniform(-3.0, 3.0, 40)
    spec[:6] = [10.0, 8.5, 7.2, 6.0, -9.0, -7.5]
    op = dict(kind=1, n=40, mat=spec, rot_seed=9)
    a = port.lanczos(op, 24, 13, k=4, l=2, workers=workers)
    b = ref.lanczos(op, 24, 13, k=4, l=2, workers=workers)
    assert (a["diag"] == b["diag"]).all() and (a["off"] == b["off"]).all()
    assert (a["eigvals"] == b["eigvals"]).all() and (a["eigvecs"] == b["eigvecs"]).all()


@pytest.mark.parametrize("trainer,base,workers,k", [("dho2", "adamw", 2, 4), ("fosi", "momentum", 1, 6),
                                                     ("sgd", "sgd", 2, 0), ("dho2", "adam", 3, 3)])
def test_train_quadratic_bitwise(port, ref, trainer, base, workers, k):
    spec = 0.5 + np.arange(12.0)
    w0 = port.rng_normal(41, 12)
    cfg = train_cfg(trainer, base_cfg(base), k=k, alpha=1.0, sigma=0.1, outer_rounds=3, inner_epochs=2, epochs=4,
                    batch_size=1, seed=15)
    a = port.train_quadratic(cfg, spec, 6, w0, workers=workers)
    b = ref.train_quadratic(cfg, spec, 6, w0, workers=workers)
    assert (a["w_final"] == b["w_final"]).all() and (a["loss"] == b["loss"]).all()
    assert np.array_equal(a["resid"], b["resid"], equal_nan=True) and a["refreshes"] == b["refreshes"]


def test_quadratic_known_answers(port):  # test_oracle.cpp:32-66
    h, v = port.quadratic_apply([4.0, 1.0], 0, [1.0, 1.0])
    assert abs(v - 2.5) <= 1e-15 and (h == [4.0, 1.0]).all()
    assert (port.quadratic_apply([4.0, 1.0], 0, [1.0, 0.0])[0] == [4.0, 0.0]).all()
    spec = 0.5 + np.arange(6.0)
    w = port.rng_normal(44, 6)
    g = port.quadratic_apply(spec, 3, w)[0]
    for i in range(6):  # gradient == central FD of value
        e = np.zeros(6)
        e[i] = 1e-5
        fd = (port.quadratic_apply(spec, 3, w + e)[1] - port.quadratic_apply(spec, 3, w - e)[1]) / 2e-5
        assert abs(g[i] - fd) <= 1e-6 * max(1.0, abs(fd))
    H = np.stack([port.quadratic_apply(spec, 3, c)[0] for c in np.eye(6)], axis=1)
    assert np.linalg.norm(H - H.T) <= 1e-12
    assert np.allclose(np.linalg.eigvalsh(H), spec, rtol=1e-10, atol=0)
    Q = port.quadratic_rotation(6, 3)
    assert np.abs(Q.T @ Q - np.eye(6)).max() <= 1e-14
    from oracle.bindings import CheckerError
    for bad in ([], [1.0, 0.0], [1.0, np.inf]):
        with pytest.raises(CheckerError):
            port.quadratic_apply(bad, 0, np.ones(len(bad)))


def test_train_quadratic_known_answers(port):  # test_trainer.cpp:47-99, :197-239
    spec = np.array([9.0, 5, 3, 2, 1, 0.5])
    w0 = port.rng_normal(8, 6)
    one = port.train_quadratic(train_cfg("fosi", base_cfg("sgd", lr=0.0), k=6, alpha=1.0, epochs=1, batch_size=1,
                                         seed=5), spec, 4, w0)
    assert len(one["loss"]) == 1 and one["loss"][0] <= 1e-12 and np.linalg.norm(one["w_final"]) <= 1e-8
    assert one["refreshes"] == 1
    spec10 = 1.0 + np.arange(10.0)
    for workers in (1, 2):
        w0 = port.rng_normal(31, 10)
        sgd = port.train_quadratic(train_cfg("sgd", base_cfg("sgd", lr=0.05), epochs=4, batch_size=1, seed=9),
                                   spec10, 2, w0, workers=workers)
        fosi = port.train_quadratic(train_cfg("fosi", base_cfg("sgd", lr=0.05), k=0, l=0, epochs=4, batch_size=1,
                                              seed=9), spec10, 2, w0, workers=workers)
        assert (sgd["w_final"] == fosi["w_final"]).all() and (sgd["loss"] == fosi["loss"]).all()
        assert fosi["refreshes"] == 0
    res = port.train_quadratic(train_cfg("dho2", base_cfg("adamw"), k=4, alpha=1.0, sigma=0.1, outer_rounds=3,
                                         inner_epochs=2, batch_size=1, seed=15), 0.5 + np.arange(12.0), 6,
                               port.rng_normal(41, 12), workers=2)
    assert len(res["loss"]) == 6 and not np.isnan(res["resid"]).any()
    from oracle.bindings import CheckerError
    with pytest.raises(CheckerError):  # a diverging run aborts (test_trainer.cpp:181-195)
        port.train_quadratic(train_cfg("sgd", base_cfg("sgd", lr=1e6), epochs=400, batch_size=1, seed=3),
                             1.0 + 10.0 * np.arange(8.0), 1, port.rng_normal(2, 8))


def test_golden_quadratic(port):
    G = np.load(os.path.join(GOLDEN, "golden.npz"))
    if "q_Q" not in G.files:
        pytest.skip("quadratic fixtures not generated")
    assert (port.quadratic_rotation(40, 9) == G["q_Q"]).all()
    hx, val = port.quadratic_apply(G["q_spec"], 9, G["q_x"])
    assert (hx == G["q_hx"]).all() and val == G["q_val"]
    a = port.lanczos(dict(kind=1, n=40, mat=G["q_spec"], rot_seed=9), 24, 13, k=4, l=2, workers=2)
    assert (a["diag"] == G["q_lz_diag"]).all() and (a["eigvecs"] == G["q_lz_eigvecs"]).all()
    cfg = train_cfg("dho2", base_cfg("adamw"), k=4, alpha=1.0, sigma=0.1, outer_rounds=3, inner_epochs=2,
                    batch_size=1, seed=15)
    t = port.train_quadratic(cfg, G["t_spec"], 6, G["t_w0"], workers=2)
    assert (t["w_final"] == G["t_wfinal"]).all() and (t["loss"] == G["t_loss"]).all()
