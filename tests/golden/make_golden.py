"""Generates tests/golden/golden.npz from the UNMODIFIED reference library (oracle/_ref/libdho2ref.so,
compiled from /root/reference/proj/src by oracle/Makefile). Run here, where the reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the CPU checker on machines without /root/reference (test_oracle_pin.py)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import CpuChecker, base_cfg, blobs_dataset, train_cfg  # noqa: E402


def main():
    R = CpuChecker("reference")
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(37, 20, 5, seed=3)
    w = R.mlp_init(sizes, 1) + 0.01 * R.rng_normal(4, R.mlp_dim(sizes))
    v = R.rng_normal(8, len(w))
    hv = R.mlp_hvp(sizes, w, v, X, y, 5)
    g = R.mlp_grad(sizes, w, X, y, 5)
    op = dict(kind=2, n=len(w), sizes=sizes, w=w, X=X, y=y, ncls=5)
    lz = R.lanczos(op, 20, 77, k=4, l=2, workers=3)
    tX, ty = blobs_dataset(200, 20, 5, seed=7)
    w0 = R.mlp_init(sizes, 2)
    cfg = train_cfg("dho2", base_cfg("momentum"), k=3, l=1, outer_rounds=2, inner_epochs=2, batch_size=16,
                    curvature_batch=40, seed=21)
    tr = R.train_mlp(cfg, sizes, tX, ty, w0, workers=2, ncls=5)
    # QuadraticOracle (oracle.cpp:233-286): rotation, apply_h / value, Lanczos and a DHO2 run on it
    q_spec = np.random.default_rng(200).uniform(-3.0, 3.0, 40)
    q_spec[:6] = [10.0, 8.5, 7.2, 6.0, -9.0, -7.5]
    q_Q = R.quadratic_rotation(40, 9)
    q_x = R.rng_normal(31, 40)
    q_hx, q_val = R.quadratic_apply(q_spec, 9, q_x)
    q_lz = R.lanczos(dict(kind=1, n=40, mat=q_spec, rot_seed=9), 24, 13, k=4, l=2, workers=2)
    t_spec = 0.5 + np.arange(12.0)
    t_w0 = R.rng_normal(41, 12)
    q_cfg = train_cfg("dho2", base_cfg("adamw"), k=4, alpha=1.0, sigma=0.1, outer_rounds=3, inner_epochs=2,
                      batch_size=1, seed=15)
    q_tr = R.train_quadratic(q_cfg, t_spec, 6, t_w0, workers=2)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, mlp_sizes=np.array(sizes), mlp_w=w, mlp_v=v, mlp_X=X, mlp_y=y, mlp_hv=hv, mlp_g=g,
                        lz_m=20, lz_seed=77, lz_diag=lz["diag"], lz_off=lz["off"], lz_eigvals=lz["eigvals"],
                        tr_X=tX, tr_y=ty, tr_w0=w0, tr_wfinal=tr["w_final"], tr_loss=tr["loss"],
                        q_spec=q_spec, q_Q=q_Q, q_x=q_x, q_hx=q_hx, q_val=q_val, q_lz_diag=q_lz["diag"],
                        q_lz_eigvals=q_lz["eigvals"], q_lz_eigvecs=q_lz["eigvecs"], t_spec=t_spec, t_w0=t_w0,
                        t_wfinal=q_tr["w_final"], t_loss=q_tr["loss"], t_resid=q_tr["resid"])
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
