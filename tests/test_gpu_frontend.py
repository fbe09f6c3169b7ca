"""A config file run end to end on the device (config.run_config -> artifacts) against the
unmodified reference harness's run_experiment on the same file.

Bit-exact: row count, epochs, outer/inner indices, refresh flags, ese_refreshes, gs_flops, the
modeled clock at one worker, D_shard slots, summary keys (ours adds "gpus"). Within the §8d
end-to-end bounds: losses (1e-4 rel for SGD / Heavy-Ball, 1e-3 for Adam-family), final params."""
import csv
import json
import os

import numpy as np
import pytest

import paper_2505_00982_b200 as d
from paper_2505_00982_b200 import artifacts as A
from paper_2505_00982_b200 import config as CF

pytestmark = pytest.mark.gpu

CONFIGS = {
    "quadratic_dho2": ("""[experiment]
trainer = dho2
seed = 3
[problem]
kind = quadratic
n = 40
condition = 1e3
rotation_seed = 5
[optimizer]
base = momentum
lr = 0.01
k = 4
alpha = 0.5
[training]
K = 2
P = 2
sigma = 0.1
batch_size = 1
""", 1e-4),
    "mlp_fosi": ("""[experiment]
trainer = fosi
seed = 2
[problem]
kind = mlp
dataset = two-gaussians
samples = 200
layers = 2, 16, 2
[optimizer]
base = adam
k = 2
l = 1
curvature_batch = 64
[training]
epochs = 3
batch_size = 16
""", 1e-3),
    "mlp_sgd_regression": ("""[experiment]
trainer = sgd
[problem]
kind = mlp
dataset = linear-regression
samples = 96
layers = 3, 8, 1
loss = mse
[optimizer]
base = sgd
lr = 0.05
[training]
epochs = 2
batch_size = 8
""", 1e-4),
}


def with_out(text, out_dir):
    """The same config with [experiment] out pointed at out_dir (the reference writes there)."""
    return text.replace("[experiment]\n", f"[experiment]\nout = {out_dir}\n", 1)


def read_metrics(path):
    with open(path) as f:
        return list(csv.DictReader(f))


@pytest.fixture(scope="module")
def harness():
    from oracle.bindings import RefHarness, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libdho2ref.so not built")
    return RefHarness()


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_run_config_matches_reference_harness(ctx, harness, tmp_path, name):
    text, tol = CONFIGS[name]
    ref_dir, our_dir = str(tmp_path / "ref"), str(tmp_path / "gpu")
    assert harness.run_experiment(with_out(text, ref_dir)) == 0
    assert CF.run_config(ctx, CF.parse_config_text(text), our_dir) == 0
    rp, op = A.RunPaths.in_dir(ref_dir), A.RunPaths.in_dir(our_dir)
    rm, om = read_metrics(rp.metrics_csv), read_metrics(op.metrics_csv)
    assert list(rm[0].keys()) == list(om[0].keys()) and len(rm) == len(om)
    for a, b in zip(rm, om):
        for key in ("trainer", "outer_k", "inner_l", "epoch", "ese_refresh_flag"):
            assert a[key] == b[key], key
        la, lb = float(a["train_loss"]), float(b["train_loss"])
        assert abs(la - lb) <= tol * max(abs(la), 1e-6)
        assert (a["train_acc"] == "") == (b["train_acc"] == "")
        assert (a["residual_norm"] == "") == (b["residual_norm"] == "")
        assert abs(float(a["wallclock_ms"]) - float(b["wallclock_ms"])) <= 1e-9 * max(float(a["wallclock_ms"]), 1.0)
    rs, os_ = json.load(open(rp.summary_json)), json.load(open(op.summary_json))
    assert set(os_) - set(rs) == {"gpus"} and set(rs) <= set(os_)
    for key in ("trainer", "workers", "n", "samples", "k", "l", "lanczos_m", "rounds_per_epoch", "epochs_run",
                "ese_refreshes", "gs_flops", "safeguard_passes", "d_shard_slots_per_rank", "aborted", "problem_kind"):
        assert rs[key] == os_[key], key
    # the reference's own memory_report reads our run exactly as it reads its own (an SGD run, which never
    # allocates a basis, is a MISMATCH in both)
    assert harness.memory_report([our_dir]) == harness.memory_report([ref_dir])
    mem = {r["object"]: int(r["peak_slots"]) for r in csv.DictReader(open(op.memory_csv))}
    ref_mem = {r["object"]: int(r["peak_slots"]) for r in csv.DictReader(open(rp.memory_csv))}
    for key in ("D_shard", "B", "h_shard", "w"):
        if key in ref_mem:
            assert mem[key] == ref_mem[key], key


def test_diverging_config_aborts_like_reference(ctx, harness, tmp_path):
    text = """[experiment]
trainer = sgd
[problem]
kind = quadratic
n = 8
condition = 1e2
[optimizer]
base = sgd
lr = 1e6
[training]
epochs = 400
batch_size = 1
"""
    ref_dir, our_dir = str(tmp_path / "ref"), str(tmp_path / "gpu")
    assert harness.run_experiment(with_out(text, ref_dir)) == 2
    assert CF.run_config(ctx, CF.parse_config_text(text), our_dir) == 2
    rs, os_ = json.load(open(A.RunPaths.in_dir(ref_dir).summary_json)), json.load(open(A.RunPaths.in_dir(our_dir).summary_json))
    assert rs["aborted"] and os_["aborted"] and "non-finite loss" in os_["abort_reason"]
