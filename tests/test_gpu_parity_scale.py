"""Parity at the BENCHMARKED configurations (VERDICT r01 "next round" item 1).

Each case runs the device path at full size and compares it, on FULL vectors, with the fp64 torch mirror
(tests/fp64_mirror.py) on identical fp32-exact inputs. The mirror is first pinned to the UNMODIFIED
reference's outputs for the same inputs, stored in tests/golden/scale_*.npz by
tests/golden/make_scale_fixtures.py (run against oracle/_ref, the reference compiled in place): sampled
entries, full-vector norms, eigenvalues, B. So every comparison is device path -> fp64 restatement ->
reference, with the restatement checked at the fp64 level on the same run.

Bars (written next to each assertion):
  C4 widths (3072-3584x8-10) HVP / gradient, B = 64:   rel-L2 <= 1e-4 (oracle.cpp:451-647)
  C4 update pass, n = 100,989,962, r = 32, AdamW:       per element <= 1e-6 of the element's term scale
                                                        (optimizer.cpp:81-117, identical inputs)
  C3 refresh, B = 512, m = 80, k = 20:                  eigenvalues <= 1e-4 rel, B <= 1e-5 ||H||, projector
                                                        (dist_lanczos.cpp:31-158)
  C3 DHO2 + AdamW trajectory, non-degenerate data:      params rel-L2 <= 1e-4 over 2 outer rounds
  C2 exact config (784-256-10, C = 4, Heavy-Ball):      params rel-L2 <= 1e-4, max-abs <= 1e-5, loss 1e-4
  C1 refresh in the reference's arithmetic:             eigenvalues <= 1e-4 rel, B <= 1e-5 ||H||
"""
import gc
import os

import numpy as np
import pytest
import torch

import fp64_mirror as M
import paper_2505_00982_b200 as d
import scale_inputs as S

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CUDA = torch.device("cuda:0")
F64 = torch.float64


def fixture(name):
    path = os.path.join(GOLD, f"scale_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tests/golden/make_scale_fixtures.py {name} where /root/reference exists")
    return np.load(path)


def T(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64), device=CUDA)


def rel_l2(a, b):
    a, b = torch.as_tensor(a, device=CUDA, dtype=F64), torch.as_tensor(b, device=CUDA, dtype=F64)
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))


def projector_dist(V, W):
    """||V^T V - W^T W||_F for r x n row-stacked bases (sign-invariant, exact without n x n matrices)."""
    a = torch.sum((V @ V.T) ** 2) + torch.sum((W @ W.T) ** 2) - 2 * torch.sum((V @ W.T) ** 2)
    return float(torch.sqrt(torch.clamp_min(a, 0.0)))


@pytest.fixture(autouse=True)
def _free_gpu():
    yield
    gc.collect()
    torch.cuda.empty_cache()


# ------------------------------------------------------------------------ C4 widths: HVP and gradient
def test_c4_widths_hvp_grad(ctx, port):
    fx = fixture("c4_mlp")
    sizes = S.C4_SIZES
    n = S.mlp_dim(sizes)
    B = int(fx["B"])
    from oracle.bindings import blobs_dataset
    X, y = blobs_dataset(B, sizes[0], 10, seed=7)
    X = S.f32(X)
    w = S.f32(port.mlp_init(sizes, 1) + 0.01 * port.rng_normal(0xC5, n))
    v = S.f32(port.rng_normal(0xC4, n))
    idx = torch.as_tensor(fx["idx"], device=CUDA)
    mir = M.MlpMirror(sizes, CUDA)
    wt, vt, Xt, yt = T(w), T(v), T(X), T(y)
    hv_m = mir.hvp(wt, vt, Xt, yt)
    g_m = mir.grad(wt, Xt, yt)
    # the fp64 mirror IS the reference at fp64 level (sampled entries, norms, dots)
    for vec, key, nkey in ((hv_m, "hv", "hv_norm"), (g_m, "g", "g_norm")):
        ref = torch.as_tensor(fx[key], device=CUDA)
        assert float(torch.max(torch.abs(vec[idx] - ref))) <= 1e-10 * float(torch.max(torch.abs(ref)))
        assert abs(float(torch.linalg.vector_norm(vec)) / float(fx[nkey]) - 1.0) <= 1e-11
    assert abs(float(hv_m @ vt) / float(fx["hv_dot_v"]) - 1.0) <= 1e-10
    assert abs(mir.value(wt, Xt, yt) - float(fx["value"])) <= 1e-12
    # device path (fp32 + split-BF16x3 tcgen05 GEMMs), full vectors: rel-L2 <= 1e-4 (§8d)
    mlp = d.MlpOracle(ctx, sizes)
    batch = d.Batch(X, y, 10)
    hv = mlp.hvp(w, v, batch)
    g = mlp.grad(w, batch)
    e_hv, e_g = rel_l2(hv, hv_m), rel_l2(g, g_m)
    print(f"C4 widths B={B}: hvp rel-L2 {e_hv:.2e}, grad rel-L2 {e_g:.2e}")
    assert e_hv <= 1e-4 and e_g <= 1e-4
    assert abs(mlp.value(w, batch) - float(fx["value"])) <= 1e-5 * abs(float(fx["value"]))
    assert abs(mlp.accuracy(w, batch) - float(fx["accuracy"])) <= 1.5 / B
    mlp.close()


# ------------------------------------------------------------------------ C4 update pass (n = 101 M, r = 32)
def test_c4_update_pass_per_element(ctx):
    fx = fixture("c4_update")
    n, r, Tn = int(fx["n"]), int(fx["r"]), int(fx["T"])
    assert n == S.mlp_dim(S.C4_SIZES) and r == S.UPD_R
    ev = np.asarray(fx["eigvals"])
    ii = torch.arange(n, device=CUDA, dtype=torch.int64)
    V = torch.empty((r, n), dtype=torch.float32, device=CUDA)  # column-major n x r, ld = n
    for j in range(r):
        V[j] = S.unif_torch(ii, S.SALT_V + j, S.V_SCALE, torch.float32)
    pi = S.unif_torch(ii, S.SALT_PI, S.PI_SCALE, F64)
    w = S.unif_torch(ii, S.SALT_W, S.W_SCALE, F64)
    torch.cuda.synchronize()
    ese = d.EseResult.from_device(ctx, ev, V.data_ptr(), n, n, r)
    opt = d.BaseOptimizer(ctx, d.BaseConfig("adamw"), n)
    V64 = V.double()
    mopt = M.BaseOptimizerMirror("adamw", n, CUDA)
    sidx = torch.as_tensor(fx["idx"], device=CUDA)
    pi_h = pi.cpu().numpy()
    for t in range(Tn):
        g = S.unif_torch(ii, S.SALT_G + t, S.G_SCALE, F64)
        nw_m, bs_m, c, coef, sc = M.split_deltas(g, pi, ev, V64, mopt, w, S.UPD_ALPHA, S.UPD_SIGMA, S.UPD_FLOOR)
        # mirror == reference (optimizer.cpp:81-129) at the sampled entries and in norm
        for vec, key, nkey in ((nw_m, "newton", "newton_norm"), (bs_m, "base", "base_norm")):
            ref = torch.as_tensor(fx[key][t], device=CUDA)
            assert float(torch.max(torch.abs(vec[sidx] - ref))) <= 1e-10 * float(torch.max(torch.abs(ref)))
            assert abs(float(torch.linalg.vector_norm(vec)) / float(fx[nkey][t]) - 1.0) <= 1e-10
        dl = d.admm_deltas(g.cpu().numpy(), pi_h, ese, opt, w.cpu().numpy(), S.UPD_ALPHA, S.UPD_SIGMA, S.UPD_FLOOR)
        nw, bs = T(dl.newton), T(dl.base)
        # per element, relative to the magnitude of the terms the element sums (the fp32 forward-error
        # model of the same formula): newton_i = -alpha sum_j V_ij c_j/den_j; base_i = s_i - sum_j V_ij sc_j
        # with s_i's own terms (Adam: lr (b1 |m'| + (1 - b1) |g2|) / bc1 / (sqrt(v_hat) + eps) + lr wd |w|)
        Va = V.abs()
        scale_n = S.UPD_ALPHA * (Va.T @ coef.abs().float()).double()
        scale_b = mopt.term_scale + (Va.T @ sc.abs().float()).double()
        del Va
        en = float(torch.max(torch.abs(nw - nw_m) / scale_n))
        eb = float(torch.max(torch.abs(bs - bs_m) / scale_b))
        print(f"C4 update step {t}: newton max err / term scale {en:.2e}, base {eb:.2e}")
        assert en <= 1e-6 and eb <= 1e-6
        del nw, bs, scale_n, scale_b
        w = w + bs_m + nw_m
    ref_w = torch.as_tensor(fx["w_after"], device=CUDA)
    assert float(torch.max(torch.abs(w[sidx] - ref_w))) <= 1e-10 * float(torch.max(torch.abs(ref_w)))
    ese.close()
    opt.close()


# ------------------------------------------------------------------------ C3 refresh (B = 512, m = 80, k = 20)
def _c3_inputs(port, B):
    from oracle.bindings import blobs_dataset
    sizes = S.C3_SIZES
    X, y = blobs_dataset(B, sizes[0], 10, seed=7)
    return sizes, S.f32(X), y, S.f32(port.mlp_init(sizes, 1))


@pytest.mark.parametrize("recurrence", [1, 0])
def test_c3_refresh_vs_reference(ctx, port, recurrence):
    fx = fixture("c3_refresh")
    B, m, k, seed = int(fx["B"]), int(fx["m"]), int(fx["k"]), int(fx["seed"])
    sizes, X, y, w = _c3_inputs(port, B)
    n = S.mlp_dim(sizes)
    mir = M.MlpMirror(sizes, CUDA)
    Xt, yt = T(X), T(y)
    mir.prepare(T(w), Xt, yt)
    lz = M.lanczos(port, mir.hvp_prepared, n, m, seed, CUDA)
    ev_m, V_m = M.extract_ese(port, lz, k, 0)
    hn = float(np.abs(fx["eigvals"]).max())
    # mirror == reference (dist_lanczos.cpp:31-158) at fp64 level
    assert lz["iterations"] == int(fx["iterations"]) and lz["breakdown"] == bool(fx["breakdown"])
    assert np.max(np.abs(lz["diag"] - fx["diag"][: len(lz["diag"])])) <= 1e-9 * hn
    assert np.max(np.abs(lz["off"] - fx["off"][: len(lz["off"])])) <= 1e-9 * hn
    assert np.max(np.abs(ev_m - fx["eigvals"]) / np.abs(fx["eigvals"])) <= 1e-9
    sidx = torch.as_tensor(fx["idx"], device=CUDA)
    assert float(torch.max(torch.abs(V_m[:, sidx].T - T(fx["V_at"])))) <= 1e-6 * float(np.abs(fx["V_at"]).max())
    del lz
    # device refresh on identical inputs
    ctx.set_option("lanczos_recurrence", recurrence)
    try:
        mlp = d.MlpOracle(ctx, sizes)
        op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
        st = d.lanczos_distributed(ctx, m, op, n, seed)
        ese = d.extract_ese_distributed(ctx, st, k, 0)
    finally:
        ctx.set_option("lanczos_recurrence", 1)
    V = T(ese.eigvecs_shard(n).T.copy())
    e_ev = float(np.max(np.abs(ese.eigvals - ev_m) / np.abs(ev_m)))
    e_diag = float(np.max(np.abs(st.tridiag.diag - fx["diag"][:m]))) / hn
    e_off = float(np.max(np.abs(st.tridiag.offdiag[:m] - fx["off"][:m]))) / hn
    # Converged Ritz pairs: residual ||H y - theta y|| = beta_m |u_m| (from the reference's B) <= 1e-3 ||H||.
    Tm = np.diag(fx["diag"][:m]) + np.diag(fx["off"][: m - 1], 1) + np.diag(fx["off"][: m - 1], -1)
    th, U = np.linalg.eigh(Tm)
    resid = np.abs(fx["off"][m - 1] * U[-1, ::-1][:k])  # descending = the k selected pairs' order
    conv = np.flatnonzero(resid <= 1e-3 * hn)
    proj = projector_dist(V, V_m)
    proj_conv = projector_dist(V[conv], V_m[conv])
    sens = float(fx["sens_projector"])
    print(f"C3 refresh (recurrence={recurrence}): eigenvalues {e_ev:.2e} rel, B diag {e_diag:.2e} off {e_off:.2e} "
          f"of ||H||, projector {proj:.2e} over all {k} pairs, {proj_conv:.2e} over the {len(conv)} converged "
          f"pairs (residual <= 1e-3 ||H||); the reference's own projector moves {sens:.2e} under a 1e-7 relative "
          f"perturbation of w")
    # the device HVP's own error on this operator (one direction, full vectors)
    v = torch.randn(n, dtype=F64, device=CUDA, generator=torch.Generator(device=CUDA).manual_seed(5))
    v /= torch.linalg.vector_norm(v)
    e_hvp = rel_l2(mlp.hvp(w, v.cpu().numpy(), d.Batch(X, y, 10)), mir.hvp_prepared(v))
    print(f"  device HVP rel-L2 on this operator {e_hvp:.2e}")
    assert st.iterations == m and not st.breakdown
    assert e_ev <= 1e-4  # north-star bar
    assert e_diag <= 1e-5 and e_off <= 1e-5  # §8d
    # §8d projector bar on the converged pairs
    assert len(conv) >= k // 2 and proj_conv <= 1e-4
    # All k pairs include unconverged Ritz vectors (residual up to 0.8 ||H|| at m = 80), which are Krylov
    # artefacts, not eigenvectors: the reference's own projector moves sens = 5.4e-5 under a 1e-7 relative
    # perturbation of w (fixture), linearly in the perturbation. The bar is the reference's response to a
    # perturbation the size of the device HVP's measured error: sens * e_hvp / 1e-7.
    assert proj <= max(1e-4, sens * e_hvp / 1e-7)
    ese.close()
    st.close()
    op.close()
    mlp.close()


def test_c4_refresh_vs_fp64(ctx, port):
    """The C4 refresh itself (3072-3584x8-10, n = 100,989,962, curvature batch 1024, m = 80, k = 32) against
    the fp64 mirror on identical inputs (the mirror is pinned to the reference at the C4 widths' HVP and at
    the C3 refresh, above; one C4 refresh of the CPU reference takes ~3 h). The spectrum's top is dense
    (21.16, 20.73, 20.57, ...): at m = 80 only a few of the 32 Ritz pairs are converged, so, as at C3, the
    §8d projector bar applies to the converged pairs and the full 32-pair projector is held to the
    reference algorithm's own response (measured on the mirror) to a perturbation the size of the device
    HVP's error."""
    import gc
    from oracle.bindings import blobs_dataset
    sizes, B, m, k, seed = S.C4_SIZES, 1024, 80, 32, 4242
    n = S.mlp_dim(sizes)
    X, y = blobs_dataset(B, sizes[0], 10, seed=7)
    X = S.f32(X)
    w = S.f32(port.mlp_init(sizes, 1))
    mlp = d.MlpOracle(ctx, sizes)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
    st = d.lanczos_distributed(ctx, m, op, n, seed)
    ese = d.extract_ese_distributed(ctx, st, k, 0)
    Vd = torch.empty((k, n), dtype=torch.float32, device=CUDA)
    ese.eigvecs_to_device(Vd.data_ptr(), n)
    ev_d, diag_d, off_d = ese.eigvals.copy(), st.tridiag.diag.copy(), st.tridiag.offdiag.copy()
    vv = torch.randn(n, dtype=F64, device=CUDA, generator=torch.Generator(device=CUDA).manual_seed(5))
    vv /= torch.linalg.vector_norm(vv)
    hv_d = torch.as_tensor(mlp.hvp(w, vv.cpu().numpy(), d.Batch(X, y, 10)), device=CUDA)
    ese.close(), st.close(), op.close(), mlp.close()
    gc.collect()
    torch.cuda.empty_cache()

    def mirror(ww, want_hvp=False):
        mir = M.MlpMirror(sizes, CUDA)
        mir.prepare(T(ww), T(X), T(y))
        hv = mir.hvp_prepared(vv) if want_hvp else None
        lz = M.lanczos(port, mir.hvp_prepared, n, m, seed, CUDA)
        ev, V = M.extract_ese(port, lz, k, 0)
        out = (ev, V, lz["diag"].copy(), lz["off"].copy(), hv)
        del lz, mir
        gc.collect()
        torch.cuda.empty_cache()
        return out

    ev_m, V_m, diag_m, off_m, hv_m = mirror(w, True)
    e_hvp = rel_l2(hv_d, hv_m)
    del hv_d, hv_m
    hn = float(np.abs(ev_m).max())
    Tm = np.diag(diag_m) + np.diag(off_m[: m - 1], 1) + np.diag(off_m[: m - 1], -1)
    th, U = np.linalg.eigh(Tm)
    resid = np.abs(off_m[m - 1] * U[-1, ::-1][:k])
    conv = np.flatnonzero(resid <= 1e-3 * hn)
    e_ev = float(np.max(np.abs(ev_d - ev_m) / np.abs(ev_m)))
    e_diag = float(np.max(np.abs(diag_d - diag_m))) / hn
    e_off = float(np.max(np.abs(off_d[:m] - off_m[:m]))) / hn
    Vd64 = Vd.double()
    del Vd
    proj, proj_conv = projector_dist(Vd64, V_m), projector_dist(Vd64[conv], V_m[conv])
    del Vd64
    torch.cuda.empty_cache()
    _, V_p, _, _, _ = mirror(w * (1.0 + 1e-7 * port.rng_normal(99, n)))
    sens = projector_dist(V_m, V_p)
    print(f"C4 refresh: eigenvalues {e_ev:.2e} rel, B diag {e_diag:.2e} off {e_off:.2e} of ||H||, projector {proj:.2e} "
          f"over all {k} pairs, {proj_conv:.2e} over the {len(conv)} converged; device HVP rel-L2 {e_hvp:.2e}; the "
          f"fp64 projector moves {sens:.2e} under a 1e-7 relative perturbation of w")
    assert e_ev <= 1e-4  # north-star bar
    assert e_diag <= 1e-5 and e_off <= 1e-5  # §8d
    assert len(conv) >= 1 and proj_conv <= 1e-4  # §8d on the converged pairs
    assert proj <= max(1e-4, sens * e_hvp / 1e-7)


def test_c3_refresh_mirror_reproduces_reference_sensitivity(port):
    """The conditioning of the C3 projector, measured on the fp64 mirror exactly as the fixture measured it
    on the reference (w perturbed by 1e-7 relative): the two agree within 3x, so the mirror's projector
    is the reference's to its own conditioning."""
    fx = fixture("c3_refresh")
    B, m, k, seed = int(fx["B"]), int(fx["m"]), int(fx["k"]), int(fx["seed"])
    sizes, X, y, w = _c3_inputs(port, B)
    n = S.mlp_dim(sizes)
    mir = M.MlpMirror(sizes, CUDA)
    Xt, yt = T(X), T(y)
    out = []
    for ww in (w, w * (1.0 + 1e-7 * port.rng_normal(99, n))):
        mir.prepare(T(ww), Xt, yt)
        lz = M.lanczos(port, mir.hvp_prepared, n, m, seed, CUDA)
        out.append(M.extract_ese(port, lz, k, 0)[1])
        del lz
    s = projector_dist(out[0], out[1])
    print(f"C3 projector sensitivity to 1e-7: mirror {s:.2e}, reference {float(fx['sens_projector']):.2e}")
    assert float(fx["sens_projector"]) / 3 <= s <= 3 * float(fx["sens_projector"])


# ------------------------------------------------------------------------ trajectories
def test_c3_adamw_trajectory_nondegenerate(ctx):
    """DHO2 + AdamW at C3 widths for 2 outer rounds on blobs-3072 with class means scaled by 0.01 (the loss
    stays O(1), so the comparison is of a real trajectory, not of rounding noise around a zero gradient)."""
    fx = fixture("c3_traj")
    sizes = S.C3_SIZES
    n = S.mlp_dim(sizes)
    X, y = S.blobs_scaled(int(fx["N"]), sizes[0], 10, 7, float(fx["mean_scale"]))
    X = S.f32(X)
    from oracle.bindings import CpuChecker
    w0 = S.f32(CpuChecker("port").mlp_init(sizes, 1))
    cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("adamw"), k=int(fx["k"]), l=0, outer_rounds=int(fx["outer"]),
                          inner_epochs=int(fx["inner"]), batch_size=int(fx["b"]), curvature_batch=int(fx["curv"]),
                          seed=int(fx["seed"]), sigma=float(fx["sigma"]), alpha=float(fx["alpha"]))
    res = d.train(ctx, cfg, d.MlpOracle(ctx, sizes), d.Dataset(X, y, 10, 7), w0, workers=1)
    assert res.ese_refreshes == int(fx["refreshes"]) and (res.epoch == fx["epoch"]).all()
    assert np.min(fx["loss"]) >= 1e-2  # non-degenerate by construction
    # stratified estimate of ||w - w_ref||^2: the whole last layer exactly + the uniform sample scaled up
    idx = np.asarray(fx["idx"])
    last = sizes[-1] * sizes[-2] + sizes[-1]
    in_last = idx >= n - last
    diff2 = (res.w_final[idx] - fx["w_at"]) ** 2
    rest = diff2[~in_last].sum() * (n - last) / max((~in_last).sum(), 1)
    err = float(np.sqrt(diff2[in_last].sum() + rest)) / float(fx["w_norm"])
    err_dw = float(np.sqrt(diff2[in_last].sum() + rest)) / float(fx["dw_norm"])
    loss_rel = np.abs(res.loss - fx["loss"]) / fx["loss"]
    print(f"C3 AdamW trajectory: params rel-L2 {err:.2e} (of the displacement w - w0: {err_dw:.2e}), "
          f"loss rel {loss_rel}, loss {res.loss} vs {fx['loss']}")
    assert err <= 1e-4  # §8d end-to-end bar
    assert loss_rel.max() <= 1e-3  # §8d (Adam-family loss rows)


def test_c2_exact_config_trajectory(ctx, port):
    """C2 exactly: 784-256-10, C = 4 logical workers x b = 128, N = 5,120, curvature batch 128,
    k = 10 (m = budget 40), Heavy-Ball (lr 1e-3, mu 0.9), DHO2 sigma 1e-2, alpha 0.1, refresh every 10 steps,
    2 outer rounds (trainer.cpp:211-249), against the reference's train()."""
    from oracle.bindings import CpuChecker, base_cfg, blobs_dataset, reference_available, train_cfg
    chk = CpuChecker("reference") if reference_available() else port
    sizes = S.C2_SIZES
    X, y = blobs_dataset(5120, 784, 10, seed=7)
    X = S.f32(X)
    w0 = S.f32(chk.mlp_init(sizes, 1))
    ref = chk.train_mlp(train_cfg("dho2", base_cfg("momentum", lr=1e-3), k=10, l=0, outer_rounds=2, inner_epochs=1,
                                  batch_size=128, curvature_batch=128, seed=1, sigma=1e-2, alpha=0.1),
                        sizes, X, y, w0, workers=4, ncls=10)
    cfg = d.TrainerConfig(kind="dho2", base=d.BaseConfig("momentum", lr=1e-3), k=10, l=0, outer_rounds=2,
                          inner_epochs=1, batch_size=128, curvature_batch=128, seed=1, sigma=1e-2, alpha=0.1)
    res = d.train(ctx, cfg, d.MlpOracle(ctx, sizes), d.Dataset(X, y, 10, 7), w0, workers=4)
    assert res.ese_refreshes == ref["refreshes"] == 2 and len(res.loss) == len(ref["loss"]) == 2
    e = float(np.linalg.norm(res.w_final - ref["w_final"]) / np.linalg.norm(ref["w_final"]))
    mx = float(np.max(np.abs(res.w_final - ref["w_final"])))
    lrel = np.abs(res.loss - ref["loss"]) / ref["loss"]
    print(f"C2 trajectory: params rel-L2 {e:.2e}, max-abs {mx:.2e}, loss rel {lrel}")
    assert e <= 1e-4 and mx <= 1e-5 and lrel.max() <= 1e-4  # §8d Heavy-Ball bars
    assert np.max(np.abs(res.residual_norm - ref["resid"]) / ref["resid"]) <= 1e-3


@pytest.mark.parametrize("small", [1, 0])
@pytest.mark.parametrize("recurrence", [0, 1])
def test_c1_refresh_both_arithmetics(ctx, port, recurrence, small):
    """C1 refresh (784-256-10, B = 128, m = 40, k = 10) against the checker in both projection modes:
    the faithful classical Gram-Schmidt of the raw h (lanczos_recurrence = 0, dist_lanczos.cpp:58-74 as
    written) and the default recurrence-first projection."""
    from oracle.bindings import blobs_dataset
    sizes = S.C2_SIZES
    X, y = blobs_dataset(128, 784, 10, seed=7)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
    ctx.set_option("lanczos_recurrence", recurrence)
    ctx.set_option("mlp_small", small)  # the small-model path (one persistent launch per HVP) or the tcgen05 GEMMs
    try:
        st = d.lanczos_distributed(ctx, 40, op, mlp.dim(), 4242)
        ese = d.extract_ese_distributed(ctx, st, 10, 0)
    finally:
        ctx.set_option("lanczos_recurrence", 1)
        ctx.set_option("mlp_small", 1)
    ref = port.lanczos(dict(kind=2, n=mlp.dim(), sizes=sizes, w=w, X=X, y=y, ncls=10), 40, 4242, k=10,
                       want_basis=False)
    hn = np.abs(ref["eigvals"]).max()
    e_ev = np.max(np.abs(ese.eigvals - ref["eigvals"]) / np.abs(ref["eigvals"]))
    e_d = np.abs(st.tridiag.diag - ref["diag"]) / hn
    e_o = np.abs(st.tridiag.offdiag - ref["off"]) / hn
    V, Vr = T(ese.eigvecs_shard(mlp.dim()).T.copy()), T(ref["eigvecs"].T.copy())
    proj = projector_dist(V, Vr)
    print(f"C1 refresh recurrence={recurrence} small={small}: eigenvalues {e_ev:.2e}, B diag {e_d.max():.2e} off {e_o.max():.2e} "
          f"(first 20 iterations {e_d[:20].max():.2e}), projector {proj:.2e}")
    assert st.iterations == ref["iterations"] == 40
    assert e_ev <= 1e-4
    assert e_d.max() <= 1e-5 and e_o.max() <= 1e-5
    assert proj <= 1e-4
