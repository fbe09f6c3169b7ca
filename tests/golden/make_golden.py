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
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, mlp_sizes=np.array(sizes), mlp_w=w, mlp_v=v, mlp_X=X, mlp_y=y, mlp_hv=hv, mlp_g=g,
                        lz_m=20, lz_seed=77, lz_diag=lz["diag"], lz_off=lz["off"], lz_eigvals=lz["eigvals"],
                        tr_X=tX, tr_y=ty, tr_w0=w0, tr_wfinal=tr["w_final"], tr_loss=tr["loss"])
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
