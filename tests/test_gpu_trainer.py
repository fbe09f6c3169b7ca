"""End-to-end DHO2 / FOSI / first-order trajectories on the GPU against the CPU checker
(trainer.cpp:273-298 restated in oracle/dho2_oracle.c, pinned bitwise to the reference).

Bounds (≤ 2 outer rounds): params rel-L2 ≤ 1e-4; epoch loss ≤ 1e-4 rel (Heavy-Ball,
SGD) and ≤ 1e-3 rel (Adam/AdamW, which amplify fp32 noise where |g| ~ eps); bookkeeping bit-exact
(row count, epochs, refresh count)."""
import numpy as np
import pytest

import paper_2505_00982_b200 as d

pytestmark = pytest.mark.gpu


def run_pair(ctx, port, trainer, base, sizes, N, workers, b, k=3, l=1, outer=2, inner=2, epochs=3, curv=40,
             seed=21, m=0, ncls=5):
    from oracle.bindings import base_cfg, blobs_dataset, train_cfg
    X, y = blobs_dataset(N, sizes[0], ncls, seed=7)
    w0 = port.mlp_init(sizes, 2)
    ref = port.train_mlp(train_cfg(trainer, base_cfg(base), k=k, l=l, outer_rounds=outer, inner_epochs=inner,
                                   epochs=epochs, batch_size=b, curvature_batch=curv, seed=seed),
                         sizes, X, y, w0, workers=workers, ncls=ncls)
    mlp = d.MlpOracle(ctx, sizes)
    cfg = d.TrainerConfig(kind=trainer, base=d.BaseConfig(base), k=k, l=l, outer_rounds=outer, inner_epochs=inner,
                          epochs=epochs, batch_size=b, curvature_batch=curv, seed=seed, lanczos_m=m)
    res = d.train(ctx, cfg, mlp, d.Dataset(X, y, ncls, 7), w0, workers=workers)
    return res, ref


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("trainer,base,workers,loss_tol", [("dho2", "momentum", 2, 1e-4), ("dho2", "adam", 1, 1e-3),
                                                           ("dho2", "adamw", 3, 1e-3), ("fosi", "momentum", 2, 1e-4),
                                                           ("sgd", "sgd", 2, 1e-4)])
def test_trajectory_small(ctx, port, trainer, base, workers, loss_tol):
    res, ref = run_pair(ctx, port, trainer, base, [20, 16, 12, 5], 200, workers, 16)
    assert len(res.loss) == len(ref["loss"]) and (res.epoch == ref["epoch"]).all()
    assert res.ese_refreshes == ref["refreshes"]
    assert rel_l2(res.w_final, ref["w_final"]) <= 1e-4
    assert np.max(np.abs(res.loss - ref["loss"]) / np.abs(ref["loss"])) <= loss_tol
    if trainer == "dho2":
        assert np.max(np.abs(res.residual_norm - ref["resid"]) / np.maximum(ref["resid"], 1e-12)) <= 1e-2
    else:
        assert np.isnan(res.residual_norm).all()


def test_fosi_without_curvature_is_sgd(ctx):  # test_trainer.cpp:71-99 (bitwise on the device too)
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 5]
    X, y = blobs_dataset(64, 20, 5, seed=3)
    w0 = d.MlpOracle(ctx, sizes).init_params(1)
    out = []
    for kind in ("sgd", "fosi"):
        mlp = d.MlpOracle(ctx, sizes)
        cfg = d.TrainerConfig(kind=kind, base=d.BaseConfig("sgd", lr=0.05), k=0, l=0, epochs=4, batch_size=8, seed=9)
        out.append(d.train(ctx, cfg, mlp, d.Dataset(X, y, 5, 7), w0, workers=2))
    assert (out[0].w_final == out[1].w_final).all() and (out[0].loss == out[1].loss).all()
    assert out[1].ese_refreshes == 0


def test_dho2_sigma_zero_reduces_to_fosi(ctx):  # test_trainer.cpp:101-137
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 5]
    X, y = blobs_dataset(40, 20, 5, seed=3)
    w0 = d.MlpOracle(ctx, sizes).init_params(4)
    dcfg = d.TrainerConfig(kind="dho2", outer_rounds=2, inner_epochs=2, sigma_zero_reduction=True, k=3, l=1,
                           alpha=0.05, batch_size=8, seed=21, curvature_batch=40)
    rounds = (20 + 8 - 1) // 8
    fcfg = d.TrainerConfig(kind="fosi", epochs=4, refresh_interval=2 * rounds, k=3, l=1, alpha=0.05, batch_size=8,
                           seed=21, curvature_batch=40)
    a = d.train(ctx, dcfg, d.MlpOracle(ctx, sizes), d.Dataset(X, y, 5, 7), w0, workers=2)
    b = d.train(ctx, fcfg, d.MlpOracle(ctx, sizes), d.Dataset(X, y, 5, 7), w0, workers=2)
    assert (a.w_final == b.w_final).all() and (a.loss == b.loss).all() and a.ese_refreshes == b.ese_refreshes


@pytest.mark.slow
def test_trajectory_c1_shape(ctx, port):
    """C1 (784-256-10, C=1, b=128, curvature 128, k=10, m=40, Adam, dho2) on N=1280, 2 outer rounds."""
    from oracle.bindings import base_cfg, blobs_dataset, train_cfg
    sizes = [784, 256, 10]
    X, y = blobs_dataset(1280, 784, 10, seed=7)
    w0 = port.mlp_init(sizes, 1)
    ref = port.train_mlp(train_cfg("dho2", base_cfg("adam", lr=1e-3), k=10, l=0, outer_rounds=2, inner_epochs=1,
                                   batch_size=128, curvature_batch=128, seed=1, sigma=1e-2, alpha=0.1),
                         sizes, X, y, w0, workers=1, ncls=10)
    cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("adam", lr=1e-3), k=10, l=0, outer_rounds=2, inner_epochs=1,
                          batch_size=128, curvature_batch=128, seed=1, sigma=1e-2, alpha=0.1)
    tr = d.Trainer(ctx, cfg, d.MlpOracle(ctx, sizes), d.Dataset(X, y, 10, 7), w0, workers=1)
    tr.run()
    res = tr.result()
    assert len(res.loss) == len(ref["loss"]) == 2 and res.ese_refreshes == 2
    assert rel_l2(res.w_final, ref["w_final"]) <= 1e-4
    assert np.max(np.abs(res.loss - ref["loss"]) / ref["loss"]) <= 1e-3


def test_trainer_diverges_loudly(ctx):
    from oracle.bindings import blobs_dataset
    X, y = blobs_dataset(32, 8, 4, seed=1)
    mlp = d.MlpOracle(ctx, [8, 8, 4], "relu")
    cfg = d.TrainerConfig(kind="sgd", base=d.BaseConfig("sgd", lr=1e30), epochs=3, batch_size=8)
    with pytest.raises((d.TrainingDiverged, d.NumericError)):
        d.train(ctx, cfg, mlp, d.Dataset(X, y, 4, 7), mlp.init_params(1) * 10)


def test_graph_refresh_bitwise_equal_to_eager(ctx):
    """The CUDA-graph replay of the Lanczos refresh (captured on the second refresh) launches the same
    kernels as the eager path: trajectories with 4 refreshes are bitwise identical."""
    from oracle.bindings import blobs_dataset
    sizes = [24, 32, 32, 5]
    X, y = blobs_dataset(160, 24, 5, seed=4)
    w0 = d.MlpOracle(ctx, sizes).init_params(3)
    out = []
    for graphs in (0, 1):
        ctx.set_option("graphs", graphs)
        try:
            mlp = d.MlpOracle(ctx, sizes)
            cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("adam"), k=4, l=1, outer_rounds=4, inner_epochs=1,
                                  epochs=1, batch_size=16, curvature_batch=64, seed=5)
            out.append(d.train(ctx, cfg, mlp, d.Dataset(X, y, 5, 7), w0, workers=2))
        finally:
            ctx.set_option("graphs", 1)
    assert out[0].ese_refreshes == out[1].ese_refreshes == 4
    assert (out[0].w_final == out[1].w_final).all()
    assert (out[0].loss == out[1].loss).all()
    assert ctx.stat("lanczos_graph_launches") >= 2


@pytest.mark.parametrize("trainer", ["dho2", "fosi"])
def test_host_resident_matches_device_resident(ctx, trainer):
    """End-to-end mode (dataset in pinned host memory; each next batch gathered on a host thread and
    copied while the current step computes) is bitwise the device-resident run, across epoch edges."""
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(100, 20, 5, seed=7)
    w0 = d.MlpOracle(ctx, sizes).init_params(2)
    out = []
    for host in (False, True):
        mlp = d.MlpOracle(ctx, sizes)
        cfg = d.TrainerConfig(kind=trainer, base=d.BaseConfig("adam"), k=3, l=1, outer_rounds=2, inner_epochs=2,
                              epochs=3, batch_size=16, curvature_batch=40, seed=21)
        tr = d.Trainer(ctx, cfg, mlp, d.Dataset(X, y, 5, 7), w0, workers=2, host_resident=host)
        losses = []
        while not tr.stat("done"):
            tr.step(1, with_eval=True)
            losses.append(tr.last_loss())
        res = tr.result()
        out.append((res.w_final, np.array(losses), res.loss, tr.stat("h2d_bytes")))
        tr.close()
    assert (out[0][0] == out[1][0]).all() and (out[0][1] == out[1][1]).all() and (out[0][2] == out[1][2]).all()
    assert out[1][3] > 0
