"""Generates the parity-at-scale fixtures tests/golden/scale_*.npz from the UNMODIFIED reference library
(oracle/_ref/libdho2ref.so, compiled from /root/reference/proj/src by oracle/Makefile). Run here, where the
reference exists (CPU only; the C3 cases take tens of minutes each):

    make -C oracle ref
    python tests/golden/make_scale_fixtures.py c4_mlp c4_update c3_refresh c3_traj

What each fixture holds (full reference vectors are 0.08-0.8 GB, so they keep sampled entries at
`scale_inputs.sample_indices` plus full-vector norms and dot products):
  c4_mlp      MlpOracle::hvp / grad / value / accuracy (oracle.cpp:400-647) at the C4 widths
              3072-3584x8-10 (n = 100,989,962), B = 64, fp32-exact inputs.
  c4_update   two consecutive admm_deltas steps (optimizer.cpp:81-129), AdamW, n = 100,989,962, r = 32,
              hashed fp32-exact inputs (ref_deltas_hashed).
  c3_refresh  lanczos_distributed + extract_ese_distributed (dist_lanczos.cpp:31-158) at the C3 refresh:
              3072-2048-2048-10, B = 512, m = 80, k = 20; plus the same refresh with w perturbed by
              1e-7 relative, to measure the reference's own sensitivity (projector, eigenvalues, B).
  c3_traj     train() (trainer.cpp:273-298), DHO2 + AdamW at C3 widths for 2 outer rounds on a
              non-degenerate blobs-3072 (class means scaled by 0.01, loss stays ~O(1)).
"""
import ctypes as C
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.bindings import CpuChecker, base_cfg, blobs_dataset, train_cfg  # noqa: E402
import scale_inputs as S  # noqa: E402

_dp = C.POINTER(C.c_double)


def _d(a):
    return a.ctypes.data_as(_dp)


def c4_mlp(R):
    sizes = S.C4_SIZES
    n = S.mlp_dim(sizes)
    B = 64
    X, y = blobs_dataset(B, sizes[0], 10, seed=7)
    X = S.f32(X)
    w = S.f32(R.mlp_init(sizes, 1) + 0.01 * R.rng_normal(0xC5, n))
    v = S.f32(R.rng_normal(0xC4, n))
    t0 = time.time()
    hv = R.mlp_hvp(sizes, w, v, X, y, 10)
    t1 = time.time()
    g = R.mlp_grad(sizes, w, X, y, 10)
    t2 = time.time()
    val = R.mlp_value(sizes, w, X, y, 10)
    acc = R.mlp_accuracy(sizes, w, X, y, 10)
    idx = S.sample_indices(n, sizes, 1 << 14)
    print(f"c4_mlp: n={n} B={B} hvp {t1 - t0:.1f}s grad {t2 - t1:.1f}s ({R.max_threads()} threads)")
    return dict(n=n, B=B, idx=idx, hv=hv[idx], g=g[idx], hv_norm=np.linalg.norm(hv), g_norm=np.linalg.norm(g),
                hv_dot_v=hv @ v, g_dot_v=g @ v, value=val, accuracy=acc, hvp_s=t1 - t0, grad_s=t2 - t1)


def c4_update(R):
    n = S.mlp_dim(S.C4_SIZES)
    r, T = S.UPD_R, S.UPD_T
    idx = S.sample_indices(n, None, 1 << 15)
    L = R.lib
    L.ref_deltas_hashed.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, _dp, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_int64, C.c_double, C.c_int64, C.c_double, C.c_int64, C.c_double,
                                    C.c_int64, C.c_double, C.POINTER(C.c_int64), C.c_size_t, _dp, _dp, _dp, _dp, _dp]
    cfg = base_cfg("adamw")
    ev = np.ascontiguousarray(S.UPD_EIGVALS[:r])
    newton, base, wat = np.zeros(T * len(idx)), np.zeros(T * len(idx)), np.zeros(len(idx))
    sqn, sqb = np.zeros(T), np.zeros(T)
    idx64 = np.ascontiguousarray(idx, np.int64)
    t0 = time.time()
    rc = L.ref_deltas_hashed(C.addressof(cfg), n, r, _d(ev), T, S.UPD_ALPHA, S.UPD_SIGMA, S.UPD_FLOOR,
                             S.SALT_V, S.V_SCALE, S.SALT_G, S.G_SCALE, S.SALT_PI, S.PI_SCALE, S.SALT_W, S.W_SCALE,
                             idx64.ctypes.data_as(C.POINTER(C.c_int64)), len(idx), _d(newton), _d(base), _d(wat),
                             _d(sqn), _d(sqb))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    print(f"c4_update: n={n} r={r} T={T} {time.time() - t0:.1f}s")
    return dict(n=n, r=r, T=T, idx=idx, eigvals=ev, newton=newton.reshape(T, -1), base=base.reshape(T, -1),
                w_after=wat, newton_norm=np.sqrt(sqn), base_norm=np.sqrt(sqb), wall_s=time.time() - t0)


C3_REFRESH = dict(B=512, m=80, k=20, seed=4242)


def c3_refresh(R):
    sizes = S.C3_SIZES
    n = S.mlp_dim(sizes)
    p = C3_REFRESH
    X, y = blobs_dataset(p["B"], sizes[0], 10, seed=7)
    X = S.f32(X)
    w = S.f32(R.mlp_init(sizes, 1))
    op = dict(kind=2, n=n, sizes=sizes, w=w, X=X, y=y, ncls=10)
    t0 = time.time()
    a = R.lanczos(op, p["m"], p["seed"], k=p["k"], want_basis=False)
    ta = time.time() - t0
    print(f"c3_refresh: base run {ta:.0f}s, iterations {a['iterations']}", flush=True)
    # the reference's own sensitivity: the same refresh with w perturbed by 1e-7 relative
    wp = w * (1.0 + 1e-7 * R.rng_normal(99, n))
    t0 = time.time()
    b = R.lanczos(dict(op, w=wp), p["m"], p["seed"], k=p["k"], want_basis=False)
    print(f"c3_refresh: perturbed run {time.time() - t0:.0f}s", flush=True)
    V, Vp = a["eigvecs"], b["eigvecs"]
    G = V.T @ Vp
    proj = np.sqrt(max(np.sum((V.T @ V) ** 2) + np.sum((Vp.T @ Vp) ** 2) - 2 * np.sum(G ** 2), 0.0))
    cos2 = np.diag(G) ** 2 / (np.sum(V * V, 0) * np.sum(Vp * Vp, 0))
    hn = np.abs(a["eigvals"]).max()
    sens = dict(sens_projector=proj, sens_eig_rel=np.max(np.abs(a["eigvals"] - b["eigvals"]) / np.abs(a["eigvals"])),
                sens_diag=np.max(np.abs(a["diag"] - b["diag"])) / hn,
                sens_off=np.max(np.abs(a["off"] - b["off"])) / hn, sens_1mcos2=1.0 - cos2)
    print("c3_refresh sensitivity to a 1e-7 relative perturbation of w: projector %.3e, eigenvalues %.3e, "
          "B diag %.3e off %.3e of ||H||" % (proj, sens["sens_eig_rel"], sens["sens_diag"], sens["sens_off"]))
    idx = S.sample_indices(n, sizes, 1 << 13)
    return dict(n=n, idx=idx, diag=a["diag"], off=a["off"], iterations=a["iterations"], breakdown=a["breakdown"],
                eigvals=a["eigvals"], V_at=V[idx].astype(np.float32), V_colnorm=np.linalg.norm(V, axis=0),
                wall_s=ta, threads=R.max_threads(), **p, **sens)


C3_TRAJ = dict(N=5120, mean_scale=0.01, b=512, curv=512, k=20, outer=2, inner=1, seed=1, sigma=1e-2, alpha=0.1)


def c3_traj(R):
    sizes = S.C3_SIZES
    n = S.mlp_dim(sizes)
    p = C3_TRAJ
    X, y = S.blobs_scaled(p["N"], sizes[0], 10, 7, p["mean_scale"])
    X = S.f32(X)
    w0 = S.f32(R.mlp_init(sizes, 1))
    cfg = train_cfg("dho2", base_cfg("adamw"), k=p["k"], l=0, outer_rounds=p["outer"], inner_epochs=p["inner"],
                    batch_size=p["b"], curvature_batch=p["curv"], seed=p["seed"], sigma=p["sigma"], alpha=p["alpha"])
    t0 = time.time()
    tr = R.train_mlp(cfg, sizes, X, y, w0, workers=1, ncls=10)
    print(f"c3_traj: {time.time() - t0:.0f}s, loss rows {tr['loss']}", flush=True)
    idx = S.sample_indices(n, sizes, 1 << 16)
    return dict(n=n, idx=idx, w_at=tr["w_final"][idx], w_norm=np.linalg.norm(tr["w_final"]),
                dw_norm=np.linalg.norm(tr["w_final"] - w0), loss=tr["loss"], acc=tr["acc"], resid=tr["resid"],
                epoch=tr["epoch"], refreshes=tr["refreshes"], wall_s=time.time() - t0, **p)


def main():
    R = CpuChecker("reference")
    for name in sys.argv[1:] or ["c4_mlp", "c4_update", "c3_refresh", "c3_traj"]:
        out = globals()[name](R)
        path = os.path.join(HERE, f"scale_{name}.npz")
        np.savez_compressed(path, **out)
        print("wrote", path, os.path.getsize(path), "bytes", flush=True)


if __name__ == "__main__":
    main()
