"""The drop-in proven from the reference side: the UNMODIFIED reference's own train()
runs with GpuMlpOracle (integration/gpu_oracle.hpp over libdho2gpu.so) in place of MlpOracle, with 4
worker threads calling Oracle::grad / hvp concurrently, and against the same train() with MlpOracle on the
CPU; one refresh through gpu_refresh() against lanczos_distributed + extract_ese_distributed. The binary
(oracle/_ref/drop_in_train) is built by integration/Makefile where /root/reference exists.

Bars (Heavy-Ball, <= 2 outer rounds): params rel-L2 <= 1e-4, loss per epoch_end row <= 1e-4
rel, bookkeeping (rows, refreshes) exact; refresh eigenvalues <= 1e-4 rel, projector <= 1e-4."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "drop_in_train")


@pytest.mark.parametrize("workers,base", [(4, "momentum"), (2, "adamw")])
def test_reference_train_with_gpu_oracle(workers, base):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/drop_in_train not built (needs /root/reference at build time)")
    out = subprocess.run([BIN, "--workers", str(workers), "--base", base, "--outer", "2"], capture_output=True,
                         text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    print(json.dumps({k: r[k] for k in ("params_rel_l2", "params_max_abs", "refresh_eig_rel", "refresh_projector",
                                         "cpu_ms", "gpu_ms")}))
    assert r["rows"][0] == r["rows"][1] == 2 and r["refreshes"][0] == r["refreshes"][1] == 2
    assert r["params_rel_l2"] <= 1e-4
    loss_tol = 1e-4 if base == "momentum" else 1e-3  # §8d: Adam-family loss rows 1e-3
    for (lc, ac), (lg, ag) in zip(r["cpu_loss_acc"], r["gpu_loss_acc"]):
        assert abs(lg - lc) <= loss_tol * abs(lc)
    assert r["refresh_eig_rel"] <= 1e-4 and r["refresh_projector"] <= 1e-4
    assert r["vhat_rows"] == r["n"]  # the full V_hat, as extract_ese_distributed returns it
