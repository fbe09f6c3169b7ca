"""One-off parity evidence at scale (SURVEY §8d per-refresh bar, identical inputs): a C3-shaped refresh
(MLP 3072-2048-2048-10, n = 10,510,346) on the GPU against the UNMODIFIED reference library's
lanczos_distributed + extract_ese on the same w, curvature batch and seed.

    python scripts/parity_c3_refresh.py [B] [m] [k]      (defaults 256 40 20; the CPU side takes minutes)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from oracle.bindings import CpuChecker, blobs_dataset, reference_available  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    sizes = [3072, 2048, 2048, 10]
    R = CpuChecker("reference" if reference_available() else "port")
    X, y = blobs_dataset(B, 3072, 10, seed=7)
    w = R.mlp_init(sizes, 1)
    n = len(w)
    ctx = d.Context(0)
    mlp = d.MlpOracle(ctx, sizes)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 10))
    t0 = time.perf_counter()
    st = d.lanczos_distributed(ctx, m, op, n, 4242)
    ese = d.extract_ese_distributed(ctx, st, k, 0)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = R.lanczos(dict(kind=2, n=n, sizes=sizes, w=w, X=X, y=y, ncls=10), m, 4242, k=k, l=0, want_basis=False)
    t_cpu = time.perf_counter() - t0
    ev, evr = ese.eigvals, ref["eigvals"]
    V, Vr = ese.eigvecs_shard(n), ref["eigvecs"]
    proj2 = np.sum((V.T @ V) ** 2) + np.sum((Vr.T @ Vr) ** 2) - 2 * np.sum((V.T @ Vr) ** 2)
    hn = np.abs(evr).max()
    print(f"C3-shaped refresh parity: n={n} B={B} m={m} k={k}; {R.kind} library {R.max_threads()} threads "
          f"{t_cpu:.1f} s vs GPU {t_gpu * 1e3:.1f} ms (first call, incl. setup)")
    print(f"  iterations {st.iterations} vs {ref['iterations']}; breakdown {st.breakdown} vs {ref['breakdown']}")
    print(f"  B diag max |diff| / ||H|| = {np.abs(st.tridiag.diag - ref['diag']).max() / hn:.2e}  (bar 1e-5)")
    print(f"  B off  max |diff| / ||H|| = {np.abs(st.tridiag.offdiag - ref['off'][:len(st.tridiag.offdiag)]).max() / hn:.2e}")
    print(f"  eigenvalues max rel diff  = {np.max(np.abs(ev - evr) / np.abs(evr)):.2e}  (bar 1e-4)")
    print(f"  projector ||VV^T - VrVr^T||_F = {np.sqrt(max(proj2, 0.0)):.2e}  (bar 1e-4)")
    print(f"  top eigenvalues GPU {np.round(ev[:4], 6)} ref {np.round(evr[:4], 6)}")
    # where the projector difference lives: per Ritz pair, 1 - cos^2 against the reference vector and the
    # relative gap to the nearest other Ritz value (ill-separated, unconverged pairs rotate first)
    cos2 = (np.sum(V * Vr, axis=0) ** 2) / (np.sum(V * V, axis=0) * np.sum(Vr * Vr, axis=0))
    gaps = np.array([np.min(np.abs(np.delete(evr, j) - evr[j])) / hn for j in range(len(evr))])
    for j in np.argsort(cos2)[:5]:
        print(f"  pair {j:2d}: eigenvalue {evr[j]:.6f}  1-cos^2 {1 - cos2[j]:.2e}  relative gap {gaps[j]:.2e}")
    for kk in (5, 10):
        A, Ar = V[:, :kk], Vr[:, :kk]
        p2 = np.sum((A.T @ A) ** 2) + np.sum((Ar.T @ Ar) ** 2) - 2 * np.sum((A.T @ Ar) ** 2)
        print(f"  projector over the top {kk}: {np.sqrt(max(p2, 0.0)):.2e}")


if __name__ == "__main__":
    main()
