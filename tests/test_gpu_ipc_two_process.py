"""Two processes on ONE GPU: the multi-process data path without NCCL. Each rank is a
separate process with its own Context; collectives go through a gloo process group (host-transport
communicator, dho2g_comm_init_host). With hvp_route = 1 the batch-split HVP's weight-block epilogues store
straight into the owner's receive buffer, which the other process opened from a CUDA-IPC handle exchanged
over the communicator — the peer-pointer path an 8-GPU run uses over NVLink, exercised across processes
before any multi-GPU box. Compared with the single-rank run and the plain reduce-scatter path."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2505_00982_b200 as d

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_two(tmp_path, route, small):
    port = free_port()
    outs = [str(tmp_path / f"r{r}_{route}_{small}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_worker.py"), str(r), "2", str(port),
                               outs[r], str(route), str(small)], cwd=ROOT, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(2)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=300)[0].decode(errors="replace"))
        except subprocess.TimeoutExpired:
            p.kill()
            raise
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [np.load(o) for o in outs]


@pytest.mark.parametrize("small", [1, 0])
def test_ipc_routed_hvp_two_processes_one_gpu(ctx, tmp_path, small):
    from oracle.bindings import blobs_dataset
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(96, 20, 5, seed=3)
    ctx.set_option("mlp_small", small)
    try:
        mlp = d.MlpOracle(ctx, sizes)
        w = mlp.init_params(1)
        op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 5))
        st = d.lanczos_distributed(ctx, 12, op, mlp.dim(), 77)
        d1, o1 = st.tridiag.diag.copy(), st.tridiag.offdiag.copy()
        st.close()
        op.close()
        mlp.close()
    finally:
        ctx.set_option("mlp_small", 1)
    fused = run_two(tmp_path, 1, small)
    plain = run_two(tmp_path, 0, small)
    for f, p in zip(fused, plain):  # fp32 rounding drift over 12 iterations (rank-split batch sums)
        assert np.abs(f["diag"] - d1).max() <= 5e-5 * np.abs(d1).max()
        assert np.abs(f["off"] - o1).max() <= 5e-5 * np.abs(o1).max()
        assert np.abs(f["diag"] - p["diag"]).max() <= 5e-5 * np.abs(d1).max()
        assert "reduce_scatter" not in list(f["ops"]) and "barrier" in list(f["ops"])
        assert "reduce_scatter" in list(p["ops"])
    # both ranks hold the same tridiagonal matrix (rank-ordered reductions)
    assert (fused[0]["diag"] == fused[1]["diag"]).all() and (plain[0]["off"] == plain[1]["off"]).all()
