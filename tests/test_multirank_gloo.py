"""Multi-rank (N > 1) data flow of the device path, exercised on CPU with torch.distributed/gloo.

The CUDA library shards every refresh and step the same way at world > 1 (lanczos.cu,
update.cu, trainer.cu); these tests run that exact decomposition with numpy arithmetic on
world_size 2 and 3 gloo ranks and check it against the single-process CPU checker:
  * Shard::for_rank row ranges partition [0, n) (collectives.cpp:10-20), workers -> ranks;
  * Lanczos: all_gather(v_i) -> batch-split HVP + reduce-scatter -> pass-1 partial dots ->
    all_gather + ascending-rank sum -> pass-2 projection -> all_gather(||h'||^2) -> decide,
    with the lazy column normalisation (v_j = sigma_j D_j) of the device kernels;
  * the split update: P1 partial c -> gather/sum -> P2 on own rows -> sc -> P3 -> all_gather(w_a);
  * the gradient: each rank's logical workers batched, reduce-scatter = mean_gradient.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(n, world, rank):
    base = (n + world - 1) // world
    b = min(base * rank, n)
    return b, min(b + base, n)


def _allgather_vec(x, world):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [o.numpy() for o in out]


def _ordered_sum(parts):
    s = parts[0].copy()
    for p in parts[1:]:
        s = s + p  # ascending rank (collectives.cpp:310-324)
    return s


def _lanczos_rank(rank, world, port, n, m, seed, op, q):
    """Sharded Lanczos as lanczos_run_into() executes it at world > 1."""
    from oracle.bindings import CpuChecker
    P = CpuChecker("port")
    b, e = _shard(n, world, rank)
    base = (n + world - 1) // world
    D = np.zeros((base, m + 1))
    v1 = P.seeded_unit_gaussian(n, seed)  # device: counter-based SplitMix64 draw of the same stream
    raw = v1 * 1.0
    D[: e - b, 0] = raw[b:e]
    sigma = np.zeros(m + 2)
    sigma[0] = 1.0
    diag, off, iters, breakdown = np.zeros(m), np.zeros(m), m, False
    for i in range(m):
        gathered = _allgather_vec(D[:, i], world)
        vfull = np.concatenate(gathered)[:n] * sigma[i]
        if op["kind"] == "mlp":  # batch split over ranks + reduce-scatter of the partial Hv
            B = len(op["y"])
            s0, s1 = _shard(B, world, rank)
            part = np.zeros(n)
            if s1 > s0:
                part = P.mlp_hvp(op["sizes"], op["w"], vfull, op["X"][s0:s1], op["y"][s0:s1], op["ncls"]) * (
                    (s1 - s0) / B)
            t = torch.from_numpy(part)
            dist.all_reduce(t)
            h = t.numpy()[b:e]
        else:
            h = (op["H"] @ vfull)[b:e]
        hs = np.zeros(base)
        hs[: e - b] = h
        active = i + 1
        # pass 1: raw dots, ||h||^2 and the Gram column G_j = D_j^T D_i, gathered and summed in rank order
        p1 = np.concatenate([D[:, :active].T @ hs, [hs @ hs], D[:, :active].T @ D[:, i]])
        r = _ordered_sum(_allgather_vec(p1, world))
        G = r[active + 1:]
        r = r[: active + 1]
        alpha = sigma[i] * r[i]
        diag[i] = alpha
        pre = np.sqrt(r[active])
        # pass 2 coefficients: recurrence-first projection (lanczos.cu header)
        gp = np.zeros(active)
        beta_prev = off[i - 1] if i > 0 else 0.0
        if i > 0:
            gp[:i] = G_prev
            gp[i] = G[i - 1]
        c = sigma[:active] * (r[:active] - alpha * sigma[i] * G - beta_prev * sigma[i - 1] * gp * (i > 0))
        ecoef = sigma[:active] * c
        ecoef[i] += alpha * sigma[i]
        if i > 0:
            ecoef[i - 1] += beta_prev * sigma[i - 1]
        G_prev = G
        hp = hs - D[:, :active] @ ecoef
        b2 = _ordered_sum(_allgather_vec(np.array([hp @ hp]), world))[0]
        beta = np.sqrt(b2)
        if beta <= 1e-10 * pre:
            iters, breakdown = i + 1, True
            break
        off[i] = beta
        D[:, i + 1] = hp
        sigma[i + 1] = 1.0 / beta
    q.put((rank, diag[:iters], off[:iters], iters, breakdown))


def _run(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def _entry(fn, rank, world, port, q, *args):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, port, *args, q)
    finally:
        dist.destroy_process_group()


def test_shards_partition_rows():
    import paper_2505_00982_b200 as d
    for n, world in [(100989962, 8), (203530, 2), (10, 8), (7, 3)]:
        ranges = [d.shard_for_rank(n, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
    # logical workers over GPUs (trainer.cu): C=8 workers on 1/2/4/8 ranks
    for world in (1, 2, 4, 8):
        cover = sum(d.shard_for_rank(8, world, r)[1] - d.shard_for_rank(8, world, r)[0] for r in range(world))
        assert cover == 8


def _lanczos_mlp_target(rank, world, port, q):
    from oracle.bindings import CpuChecker, blobs_dataset
    P = CpuChecker("port")
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(37, 20, 5, seed=3)
    w = P.mlp_init(sizes, 1)
    _lanczos_rank(rank, world, port, len(w), 15, 77, dict(kind="mlp", sizes=sizes, w=w, X=X, y=y, ncls=5), q)


def _lanczos_dense_target(rank, world, port, q):
    from oracle.bindings import CpuChecker
    P = CpuChecker("port")
    a = P.rng_normal(901, 60 * 60).reshape(60, 60)
    H = a @ a.T
    _lanczos_rank(rank, world, port, 60, 24, 19, dict(kind="dense", H=H), q)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lanczos_matches_single_rank(port, world):
    from oracle.bindings import blobs_dataset
    out = _run(_lanczos_mlp_target, world)
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(37, 20, 5, seed=3)
    w = port.mlp_init(sizes, 1)
    ref = port.lanczos(dict(kind=2, n=len(w), sizes=sizes, w=w, X=X, y=y, ncls=5), 15, 77, workers=1)
    for rank, diag, off, iters, bd in out:
        assert iters == ref["iterations"] and bd == ref["breakdown"]
        assert np.max(np.abs(diag - ref["diag"])) <= 1e-10 * np.max(np.abs(ref["diag"]))
        assert np.max(np.abs(off - ref["off"])) <= 1e-10 * np.max(np.abs(ref["off"]))
    # every rank holds the bitwise-identical B (replicated eigensolve)
    assert all((o[1] == out[0][1]).all() and (o[2] == out[0][2]).all() for o in out)


def test_sharded_lanczos_dense_uneven(port):
    out = _run(_lanczos_dense_target, 3)
    a = port.rng_normal(901, 60 * 60).reshape(60, 60)
    ref = port.lanczos(dict(kind=0, n=60, mat=a @ a.T), 24, 19, workers=1)
    for rank, diag, off, iters, bd in out:
        assert iters == ref["iterations"]
        assert np.max(np.abs(diag - ref["diag"]) / np.abs(ref["diag"]).max()) <= 1e-10


def _update_target(rank, world, port, q):
    """split_update() at world > 1: P1 partials -> ordered sum -> P2 on own rows -> sc -> P3."""
    from oracle.bindings import CpuChecker
    P = CpuChecker("port")
    n, r = 1001, 4
    V = np.linalg.qr(P.rng_normal(1, n * r).reshape(n, r))[0]
    ev = np.array([5.0, 2.0, 1e-9, -1.0])
    g, pi, w = P.rng_normal(2, n), P.rng_normal(3, n), P.rng_normal(4, n)
    alpha, sigma, lr, fl = 0.3, 0.05, 1e-2, 1e-6
    b, e = _shard(n, world, rank)
    Vs, gt = V[b:e], g[b:e] + pi[b:e]
    c = _ordered_sum(_allgather_vec(Vs.T @ gt, world))
    g2 = gt - Vs @ c
    s = -lr * g2  # sgd base step (momentum/adam state is row-local and needs no exchange)
    sc = _ordered_sum(_allgather_vec(Vs.T @ s, world))
    den = np.where(ev == 0, fl, np.sign(ev) * np.maximum(np.abs(ev), fl)) + sigma
    den = np.where(np.abs(den) < fl, np.where(den < 0, -fl, fl), den)
    base = s - Vs @ sc
    newton = -Vs @ (alpha * c / den)
    w_new = w[b:e] + base + newton
    full = np.concatenate(_allgather_vec(np.pad(w_new, (0, (n + world - 1) // world - (e - b))), world))[:n]
    q.put((rank, full))


def test_sharded_update_matches_checker(port):
    from oracle.bindings import base_cfg
    out = _run(_update_target, 2)
    n, r = 1001, 4
    V = np.linalg.qr(port.rng_normal(1, n * r).reshape(n, r))[0]
    g, pi, w = port.rng_normal(2, n), port.rng_normal(3, n), port.rng_normal(4, n)
    _, _, w_ref = port.deltas_seq(base_cfg("sgd", lr=1e-2), np.array([5.0, 2.0, 1e-9, -1.0]), V, g[None, :], w, 0.3,
                                  pi=pi, sigma=0.05, advance=True)
    for rank, full in out:
        assert np.max(np.abs(full - w_ref)) <= 1e-12 * np.max(np.abs(w_ref))


def _grad_target(rank, world, port, q):
    """mean_gradient at world > 1: rank's workers batched, reduce-scatter, 1/(bC) folded."""
    from oracle.bindings import CpuChecker, blobs_dataset
    P = CpuChecker("port")
    sizes = [20, 16, 5]
    N, C, b = 200, 4, 8
    X, y = blobs_dataset(N, 20, 5, seed=7)
    w = P.mlp_init(sizes, 2)
    perm = P.epoch_permutation(N, 7, 0)
    c0, c1 = _shard(C, world, rank)
    idx = []
    for c in range(c0, c1):
        sb, se = _shard(N, C, c)
        idx += [int(perm[sb + (0 * b + j) % (se - sb)]) for j in range(b)]
    part = np.zeros(len(w))
    if idx:
        part = P.mlp_grad(sizes, w, X[idx], y[idx], 5) * (len(idx) / (b * C))
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    q.put((rank, t.numpy()))


def test_sharded_gradient_matches_mean_gradient(port):
    from oracle.bindings import base_cfg, blobs_dataset, train_cfg
    out = _run(_grad_target, 2)
    sizes = [20, 16, 5]
    X, y = blobs_dataset(200, 20, 5, seed=7)
    w = port.mlp_init(sizes, 2)
    # reference: 4 simulated workers' mean gradient (trainer.cpp:92-103) via one SGD step with lr = 1
    cfg = train_cfg("sgd", base_cfg("sgd", lr=1.0), epochs=1, batch_size=8, seed=1)
    perm = port.epoch_permutation(200, 7, 0)
    gs = []
    for c in range(4):
        sb, se = _shard(200, 4, c)
        idx = [int(perm[sb + j % (se - sb)]) for j in range(8)]
        gs.append(port.mlp_grad(sizes, w, X[idx], y[idx], 5))
    g_ref = _ordered_sum(gs) * (1.0 / 4)
    for rank, g in out:
        assert np.max(np.abs(g - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))
    del cfg
