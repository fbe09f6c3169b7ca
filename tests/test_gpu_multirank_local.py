"""The multi-rank (G > 1) device path run for real on one GPU: 2 and 3 ranks, each a Context driven by
its own host thread, joined by the in-process fabric (dho2g_comm_init_local) instead of NCCL. Every
collective is a host rendezvous plus stream-ordered copies between the ranks' buffers (events only: no
kernel waits on another rank). This exercises the CUDA code's sharding — row ranges, padded all-gathers,
the HVP batch split + reduce-scatter, the GS partial all-reduces, the sharded Ritz vectors and sign argmax,
the sharded update, the trainer's gradient reduce-scatter and parameter all-gather — against the same
computation at G = 1. Reductions run in a different order than at G = 1 (rank-ordered fp64 sums, fp32
reduce-scatter), so results agree to fp32 rounding, not bitwise."""
import threading

import numpy as np
import pytest

import paper_2505_00982_b200 as d

pytestmark = pytest.mark.gpu


def run_ranks(world, fn):
    fab = d.LocalFabric(world)
    out, errs = [None] * world, []

    def worker(r):
        c = d.Context(0)
        try:
            c.comm_init_local(fab, r)
            out[r] = fn(c, r)
        except Exception as e:  # surfaced below
            errs.append(e)
        finally:
            c.close()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    fab.close()
    if errs:
        raise errs[0]
    return out


def lanczos_on(make_op, n, m, k, l, seed):
    def fn(ctx, rank):
        op = make_op(ctx)
        st = d.lanczos_distributed(ctx, m, op, n, seed)
        ese = d.extract_ese_distributed(ctx, st, k, l)
        b, e = d.shard_for_rank(n, ctx.world, rank)
        return st.tridiag.diag.copy(), st.tridiag.offdiag.copy(), ese.eigvals.copy(), ese.eigvecs_shard(e - b), \
            ctx.ledger()
    return fn


@pytest.mark.parametrize("world", [2, 3])
def test_lanczos_diag_sharded(world):
    n, m = 50_003, 30
    spec = 1.0 + (np.arange(n) % 997) * 0.01
    spec[:3] = [40.0, 30.0, -5.0]
    fn = lanczos_on(lambda c: d.diagonal_operator(c, spec), n, m, 3, 2, 11)
    (d1, o1, e1, v1, _), = run_ranks(1, fn)
    outs = run_ranks(world, fn)
    for dg, of, ev, _, ledger in outs:
        assert np.abs(dg - d1).max() <= 1e-5 * 40 and np.abs(of - o1).max() <= 1e-5 * 40
        assert np.abs(ev - e1).max() <= 1e-5 * 40
        assert {r[1] for r in ledger} >= {"all_gather", "all_reduce"}
    V = np.concatenate([o[3] for o in outs], axis=0)  # row shards in rank order
    G = V.T @ v1  # sign-invariant: matching Ritz vectors have |cos| = 1
    assert np.abs(np.abs(np.diag(G)) - 1).max() <= 1e-4


@pytest.mark.parametrize("world", [2, 3])
def test_lanczos_mlp_sharded(world):
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(37, 20, 5, seed=3)

    def make(c):
        mlp = d.MlpOracle(c, sizes)
        w = mlp.init_params(1)
        make.keep = mlp
        return d.mlp_hvp_operator(c, mlp, w, d.Batch(X, y, 5))

    nparam = sum(sizes[i] * sizes[i + 1] + sizes[i + 1] for i in range(len(sizes) - 1))
    fn = lanczos_on(make, nparam, 20, 4, 2, 77)
    (d1, o1, e1, v1, _), = run_ranks(1, fn)
    for dg, of, ev, _, ledger in run_ranks(world, fn):
        scale = np.abs(e1).max()
        assert np.abs(dg - d1).max() <= 1e-5 * scale and np.abs(ev - e1).max() <= 1e-5 * scale
        assert "reduce_scatter" in {r[1] for r in ledger}  # batch-split HVP partials


@pytest.mark.parametrize("world", [2, 3])
def test_ese_gather_full_vhat_on_every_rank(world):
    """dho2g_ese_gather: every rank receives the whole V_hat, as extract_ese_distributed's gather_rows
    does (dist_lanczos.cpp:148-156), equal to the 1-rank V_hat to fp32 rounding (same signs)."""
    n, m = 40_009, 24
    spec = 1.0 + (np.arange(n) % 991) * 0.01
    spec[:3] = [30.0, 20.0, -4.0]

    def fn(c, rank):
        st = d.lanczos_distributed(c, m, d.diagonal_operator(c, spec), n, 5)
        ese = d.extract_ese_distributed(c, st, 3, 1)
        return ese.eigvecs_full(n)

    (v1,), outs = run_ranks(1, fn), run_ranks(world, fn)
    for V in outs:
        assert V.shape == (n, 4)
        assert np.abs(V - v1).max() <= 1e-4 * np.abs(v1).max()
    assert all(np.array_equal(outs[0], V) for V in outs[1:])  # the same bits on every rank


def test_lanczos_rotated_quadratic_sharded():
    spec = np.linspace(-3.0, 9.0, 300)  # (no zero entry: the constructor rejects one)
    fn = lanczos_on(lambda c: d.quadratic_operator(c, spec, 5), 300, 24, 3, 1, 4)
    (d1, o1, e1, _, _), = run_ranks(1, fn)
    for dg, of, ev, _, _ in run_ranks(2, fn):
        assert np.abs(dg - d1).max() <= 1e-5 * 9 and np.abs(ev - e1).max() <= 1e-5 * 9


@pytest.mark.parametrize("world,trainer,base", [(2, "dho2", "adamw"), (3, "fosi", "momentum"), (2, "sgd", "sgd")])
def test_trainer_sharded(world, trainer, base):
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(160, 20, 5, seed=7)

    def fn(c, rank):
        mlp = d.MlpOracle(c, sizes)
        w0 = mlp.init_params(2)
        cfg = d.TrainerConfig(kind=trainer, base=d.BaseConfig(base), k=3, l=1, outer_rounds=2, inner_epochs=2,
                              epochs=3, batch_size=8, curvature_batch=40, seed=21)
        res = d.train(c, cfg, mlp, d.Dataset(X, y, 5, 7), w0, workers=4)
        return res.w_final, res.loss, res.ese_refreshes, len(c.ledger())

    (w1, l1, r1, n1), = run_ranks(1, fn)
    assert n1 == 0  # one GPU: no communication rounds
    for w, loss, refr, nrows in run_ranks(world, fn):
        assert refr == r1 and len(loss) == len(l1) and nrows > 0
        assert np.linalg.norm(w - w1) / np.linalg.norm(w1) <= 1e-5
        assert np.abs(loss - l1).max() <= 1e-4 * np.abs(l1).max()


def test_comm_ledger_report_two_ranks(tmp_path):
    """The ledger of a 2-rank device run (artifacts.run_experiment) satisfies the device comm_report: GS
    partial and beta all-reduces per iteration and pass, traffic conserved, plus the reference-schema
    memory accounting (D_shard = ceil(n/G)(m+1))."""
    from oracle.bindings import blobs_dataset
    from paper_2505_00982_b200 import artifacts as A
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(160, 20, 5, seed=7)

    def fn(c, rank):
        mlp = d.MlpOracle(c, sizes)
        cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("adam"), k=3, l=1, outer_rounds=2, inner_epochs=1,
                              batch_size=8, curvature_batch=40, seed=21)
        out = str(tmp_path / f"rank{rank}")
        rc = A.run_experiment(c, cfg, mlp, d.Dataset(X, y, 5, 7), mlp.init_params(2), out, workers=4)
        return rc, out

    outs = run_ranks(2, fn)
    for rc, out in outs:
        assert rc == 0
        rep = A.comm_report(out)
        assert "communication ledger: OK" in rep, rep
        assert "memory accounting: OK" in A.memory_report([out])


def test_seed_mismatch_is_divergence_error():
    """test_dist_lanczos.cpp:123-138: ranks that disagree on the Lanczos seed fail with DivergenceError."""
    spec = 1.0 + np.arange(1000) * 0.01

    def fn(c, rank):
        op = d.diagonal_operator(c, spec)
        try:
            d.lanczos_distributed(c, 10, op, 1000, 7 + rank)
        except d.DivergenceError as e:
            return str(e)
        return "no error"

    assert all("seed mismatch" in r for r in run_ranks(2, fn))


def test_lanczos_uneven_and_empty_shards():
    """Shard::for_rank leaves trailing ranks empty (collectives.cpp:10-20): n = 7 over 5 ranks is 2,2,2,1,0."""
    n, m = 7, 5
    spec = np.array([5.0, 4.0, 3.0, 2.0, 1.0, 0.5, -1.0])
    fn = lanczos_on(lambda c: d.diagonal_operator(c, spec), n, m, 2, 1, 3)
    (d1, o1, e1, v1, _), = run_ranks(1, fn)
    outs = run_ranks(5, fn)
    assert [o[3].shape[0] for o in outs] == [2, 2, 2, 1, 0]
    for dg, of, ev, _, _ in outs:
        assert np.abs(dg - d1).max() <= 1e-5 * 5 and np.abs(ev - e1).max() <= 1e-5 * 5
    V = np.concatenate([o[3] for o in outs], axis=0)
    assert np.abs(np.abs(np.diag(V.T @ v1)) - 1).max() <= 1e-4


def test_quadratic_trainer_with_empty_shard():
    """A rotated-quadratic DHO2 run over 4 ranks with n = 6 (shards 2,2,2,0) against 1 rank."""
    spec = np.array([9.0, 5.0, 3.0, 2.0, 1.0, 0.5])

    def fn(c, rank):
        q = d.QuadraticOracle(c, spec, 4)
        w0 = np.linspace(-1.0, 1.5, 6)
        cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("momentum", lr=0.05), k=3, alpha=0.5, sigma=0.1,
                              outer_rounds=3, inner_epochs=2, batch_size=1, seed=5)
        res = d.train(c, cfg, q, d.Dataset.dummy(4), w0, workers=4)
        q.close()
        return res.w_final, res.loss

    (w1, l1), = run_ranks(1, fn)
    for w, loss in run_ranks(4, fn):
        assert np.abs(w - w1).max() <= 1e-5 * np.abs(w1).max() and np.abs(loss - l1).max() <= 1e-5 * l1.max()


@pytest.mark.parametrize("world,B", [(2, 37), (3, 37), (3, 2)])
def test_fused_hvp_reduce_scatter(world, B):
    """hvp_route = 1: the batch-split HVP's weight-block GEMM epilogues store each element straight into
    its owner's receive slot (peer memory; one address space on the fabric), biases are routed by copies,
    and each owner sums its slots in rank order after a barrier — no reduce-scatter. B = 2 over 3 ranks
    leaves one rank with an empty batch slice (it routes zeros)."""
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(B, 20, 5, seed=3)
    nparam = sum(sizes[i] * sizes[i + 1] + sizes[i + 1] for i in range(len(sizes) - 1))

    def make(route):
        def fn(c, rank):
            c.set_option("hvp_route", route)
            mlp = d.MlpOracle(c, sizes)
            w = mlp.init_params(1)
            op = d.mlp_hvp_operator(c, mlp, w, d.Batch(X, y, 5))
            st = d.lanczos_distributed(c, 12, op, nparam, 77)
            return st.tridiag.diag.copy(), st.tridiag.offdiag.copy(), [r[1] for r in c.ledger()]
        return fn

    (d1, o1, _), = run_ranks(1, make(0))
    plain = run_ranks(world, make(0))
    fused = run_ranks(world, make(1))
    for (dg, of, ops), (dp, op_, ops_plain) in zip(fused, plain):  # fp32 rounding drift over 12 iterations
        assert np.abs(dg - d1).max() <= 5e-5 * np.abs(d1).max() and np.abs(of - o1).max() <= 5e-5 * np.abs(o1).max()
        assert np.abs(dg - dp).max() <= 5e-5 * np.abs(d1).max()
        assert "reduce_scatter" not in ops and "barrier" in ops and "reduce_scatter" in ops_plain


@pytest.mark.parametrize("world", [2, 3])
def test_trainer_fused_reduce_scatter(world):
    """hvp_route = 1 for the whole trainer: the refresh's HVPs and every step's gradient store their partials
    straight into the owners' slots (no reduce-scatter); the trajectory matches the 1-rank run."""
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(160, 20, 5, seed=7)

    def fn(c, rank):
        c.set_option("hvp_route", 1)
        mlp = d.MlpOracle(c, sizes)
        cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("adamw"), k=3, l=1, outer_rounds=2, inner_epochs=2,
                              batch_size=8, curvature_batch=40, seed=21)
        res = d.train(c, cfg, mlp, d.Dataset(X, y, 5, 7), mlp.init_params(2), workers=4)
        return res.w_final, res.loss, {r[1] for r in c.ledger()}

    (w1, l1, _), = run_ranks(1, fn)
    for w, loss, ops in run_ranks(world, fn):
        assert "reduce_scatter" not in ops and "barrier" in ops
        assert np.linalg.norm(w - w1) / np.linalg.norm(w1) <= 1e-5
        assert np.abs(loss - l1).max() <= 1e-4 * np.abs(l1).max()


def test_debug_hash_checks_two_ranks():
    """DistLanczosOptions.hash_checks / extract hash_check / TrainerConfig.debug_hash_checks
    (dist_lanczos.cpp:104-134, trainer.cpp:157): the replicated B and parameters hash equal on every rank, so
    the checks pass; with the test hook (option hash_checks = 2: ranks > 0 perturb their hash) each check
    raises the reference's DivergenceError."""
    import ctypes as C
    from paper_2505_00982_b200 import _lib as L
    from paper_2505_00982_b200.api import check
    n, m = 20_011, 12
    spec = 1.0 + (np.arange(n) % 97) * 0.1

    def fn(c, rank):
        op = d.diagonal_operator(c, spec)
        st = d.lanczos_distributed(c, m, op, n, 5, d.DistLanczosOptions(hash_checks=True))
        ese = d.extract_ese_distributed(c, st, 3, 0, hash_check=True)
        msgs = []
        c.set_option("hash_checks", 2)  # (the Python wrappers reset the option: call the C ABI directly)
        try:
            lo = L.LanczosOpts(1, 1e-6, 1e-10)
            for call in (lambda h: L.lib.dho2g_lanczos_run(c.h, op.h, m, 5, C.byref(lo), C.byref(h)),
                         lambda h: L.lib.dho2g_extract_ese(c.h, st.h, 3, 0, C.byref(h))):
                h = C.c_void_p()
                try:
                    check(call(h))
                except d.DivergenceError as e:
                    msgs.append(str(e))
        finally:
            c.set_option("hash_checks", 0)
        return st.iterations, ese.eigvals.copy(), msgs

    out = run_ranks(2, fn)
    assert out[0][0] == out[1][0] == m
    assert (out[0][1] == out[1][1]).all()
    for _, _, msgs in out:
        assert len(msgs) == 2
        assert "B diverged across ranks" in msgs[0] and "B differs across ranks" in msgs[1]


@pytest.mark.parametrize("kind", ["dho2", "sgd"])
def test_trainer_debug_hash_checks_two_ranks(kind):
    from oracle.bindings import blobs_dataset
    sizes = [12, 10, 3]
    X, y = blobs_dataset(96, 12, 3, seed=2)

    def fn(c, rank, hook):
        mlp = d.MlpOracle(c, sizes)
        w = mlp.init_params(1)
        cfg = d.TrainerConfig(kind=kind, base=d.BaseConfig("adam"), k=3, l=0, outer_rounds=2, inner_epochs=1,
                              epochs=2, batch_size=16, curvature_batch=32, seed=3, debug_hash_checks=True)
        tr = d.Trainer(c, cfg, mlp, d.Dataset(X, y, 3, 7), w, workers=2)
        if hook:
            c.set_option("hash_checks", 2)
        try:
            tr.run()
            return tr.params().copy()
        except d.DivergenceError as e:
            return str(e)
        finally:
            c.set_option("hash_checks", 0)

    out = run_ranks(2, lambda c, r: fn(c, r, False))
    assert (out[0] == out[1]).all()
    out = run_ranks(2, lambda c, r: fn(c, r, True))
    # (the refresh's B check comes first in a DHO2 run; a first-order run reaches the epoch-end parameter check)
    want = "diverged across ranks" if kind == "dho2" else "parameter replicas diverged at epoch"
    assert all(isinstance(o, str) and want in o for o in out)
