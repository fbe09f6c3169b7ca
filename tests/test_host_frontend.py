"""Config front end and run artifacts against the UNMODIFIED reference
harness (harness.cpp, compiled into oracle/_ref/libdho2ref.so): the KvConfig grammar and its error
messages, build_problem's data and w0 (bit-exact), the synthetic datasets and the CSV loader, and
the artifact writers / memory report. CPU only (no device calls)."""
import json
import os

import numpy as np
import pytest

from paper_2505_00982_b200 import artifacts as A
from paper_2505_00982_b200 import config as CF
from paper_2505_00982_b200.api import ArgumentError, TrainResult

KINDS = {0: "sgd", 1: "fosi", 2: "dho2"}
BASES = {0: "sgd", 1: "momentum", 2: "adam", 3: "adamw"}

VALID = [
    "",
    "# only a comment\n\n",
    """[experiment]
trainer = fosi   # inline comment
workers = 3
seed = 42
schedule = round_robin
out = runs/a
[problem]
kind = mlp
dataset = linear-regression
samples = 64
dataset_seed = 11
layers = 3, 8 ,1
activation = relu
loss = mse
[optimizer]
base = adam
lr = 1e-2
weight_decay = 0
beta1 = .8
beta2 = 0.99
eps = 1e-7
momentum = 0.5
k = 4
l = 2
alpha = 0.25
eigval_floor = 1e-5
refresh_interval = 7
curvature_batch = 32
[training]
epochs = 9
K = 3
P = 2
sigma = 0.125
batch_size = 8
loss_target = 1e-3
sigma_zero_reduction = true
debug_hash_checks = 1
[lanczos]
reorth_safeguard = false
safeguard_ratio = 1e-5
breakdown_rtol = 1e-9
[model]
bandwidth_gbps = 25
gflops = 2.5
""",
    """[problem]
kind = quadratic
n = 40
condition = 1e6
rotation_seed = 0
spectrum = 3, 2, 1
feature_cols = a, b,
[training]
sigma_preset = resnet-101
""",
    """  [ training ]  \n\tsigma_preset = vgg-16\nsigma = 3\n""",
]

INVALID = [
    "[experiment]\nbogus = 1\n",
    "[experiment\ntrainer = sgd\n",
    "[experiment]\ntrainer\n",
    "[experiment]\n = 3\n",
    "[experiment]\nworkers = -1\n",
    "[experiment]\nworkers = 0\n",
    "[experiment]\nseed = 1.5\n",
    "[optimizer]\nlr = fast\n",
    "[optimizer]\nlr = +1\n",
    "[optimizer]\nbase = lion\n",
    "[training]\nsigma_zero_reduction = yes\n",
    "[training]\nsigma_preset = bert\n",
    "[lanczos]\nreorth_safeguard = 2\n",
    "[problem]\nlayers = 2, x, 2\n",
    "x = 1\n",
    "[model]\nflops = 3\n",
]


def ours_as_ref_json(cfg):
    t = CF.build_trainer_config(cfg) if cfg.trainer in KINDS.values() else None
    p = cfg.problem
    out = dict(trainer=cfg.trainer, workers=cfg.workers, seed=cfg.seed, schedule=cfg.schedule, out_dir=cfg.out_dir,
               loss_target=cfg.loss_target,
               problem=dict(kind=p.kind, n=p.n, condition=p.condition, rotation_seed=p.rotation_seed,
                            spectrum=p.spectrum, dataset=p.dataset, csv_path=p.csv_path, label_col=p.label_col,
                            feature_cols=p.feature_cols, samples=p.samples, dataset_seed=p.dataset_seed,
                            layers=p.layers, activation=p.activation, loss=p.loss))
    b = t.base
    out["train"] = dict(kind={v: k for k, v in KINDS.items()}[t.kind], base_kind={v: k for k, v in BASES.items()}[b.kind],
                        lr=b.lr, weight_decay=b.weight_decay, beta1=b.beta1, beta2=b.beta2, eps=b.eps,
                        momentum=b.momentum, k=t.k, l=t.l, alpha=t.alpha, eigval_floor=t.eigval_floor,
                        refresh_interval=t.refresh_interval, curvature_batch=t.curvature_batch,
                        reorth_safeguard=t.lanczos.reorth_safeguard, safeguard_ratio=t.lanczos.safeguard_ratio,
                        breakdown_rtol=t.lanczos.breakdown_rtol, sigma=t.sigma, outer_rounds=t.outer_rounds,
                        inner_epochs=t.inner_epochs, sigma_zero_reduction=t.sigma_zero_reduction, epochs=t.epochs,
                        batch_size=t.batch_size, seed=t.seed, debug_hash_checks=t.debug_hash_checks,
                        model_bandwidth_gbps=t.model_bandwidth_gbps, model_gflops=t.model_gflops)
    return out


@pytest.fixture(scope="module")
def harness():
    from oracle.bindings import RefHarness, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libdho2ref.so not built")
    return RefHarness()


@pytest.mark.parametrize("i", range(len(VALID)))
def test_parse_matches_reference(harness, i):
    want = harness.parse_config(VALID[i], "cfg.ini")
    got = ours_as_ref_json(CF.parse_config_text(VALID[i], "cfg.ini"))
    assert got == want


@pytest.mark.parametrize("i", range(len(INVALID)))
def test_parse_errors_match_reference(harness, i):
    from oracle.bindings import CheckerError
    with pytest.raises(CheckerError) as ref_err:
        harness.parse_config(INVALID[i], "cfg.ini")
    with pytest.raises(ArgumentError) as our_err:
        CF.parse_config_text(INVALID[i], "cfg.ini")
    assert str(our_err.value) == str(ref_err.value).split("] ", 1)[1]


def test_lanczos_m_extension():
    cfg = CF.parse_config_text("[optimizer]\nk = 32\n[lanczos]\nm = 80\n")
    assert CF.build_trainer_config(cfg).lanczos_m == 80


PROBLEMS = [
    "[experiment]\nseed = 5\nworkers = 3\n[problem]\nkind = quadratic\nn = 12\n",
    "[experiment]\nseed = 2\n[problem]\nkind = quadratic\nn = 64\ncondition = 1e8\nrotation_seed = 4\n",
    "[problem]\nkind = quadratic\nspectrum = 4, 1, 0.5e-1\n",
    "[experiment]\nseed = 9\n[problem]\nkind = mlp\ndataset = concentric-rings\nsamples = 50\nlayers = 2, 8, 2\n",
    "[problem]\nkind = mlp\ndataset = two-gaussians\nsamples = 33\nlayers = 2, 5, 4, 2\nactivation = relu\n",
    "[problem]\nkind = mlp\ndataset = linear-regression\nsamples = 20\nlayers = 3, 6, 1\nloss = mse\n",
]


@pytest.mark.parametrize("i", range(len(PROBLEMS)))
def test_problem_data_bitwise(harness, i):
    want = harness.build_problem(PROBLEMS[i])
    got = CF.problem_data(CF.parse_config_text(PROBLEMS[i]))
    assert np.array_equal(got.w0, want["w0"])
    assert np.array_equal(got.dataset.features, want["X"]) and np.array_equal(got.dataset.labels, want["y"])
    assert got.dataset.n_classes == want["n_classes"]


def test_problem_errors(harness):
    from oracle.bindings import CheckerError
    for text in ("[problem]\nkind = cubic\n", "[problem]\nkind = quadratic\nn = 1\n",
                 "[problem]\nkind = mlp\nlayers = 3, 4, 2\n", "[problem]\nkind = mlp\nlayers = 2, 2\n",
                 "[problem]\nkind = mlp\ndataset = spirals\n", "[problem]\nkind = quadratic\nspectrum = 1, 0\n"):
        with pytest.raises(CheckerError) as ref_err:
            harness.build_problem(text)
        with pytest.raises(ArgumentError) as our_err:
            CF.problem_data(CF.parse_config_text(text))
        assert str(our_err.value) == str(ref_err.value).split("] ", 1)[1]


def test_synthetic_and_csv_bitwise(harness, tmp_path):
    for kind in ("two-gaussians", "concentric-rings", "linear-regression"):
        for n, seed in ((1, 0), (17, 7), (400, 123456789)):
            X, y, ncls = harness.synthetic_dataset(kind, n, seed)
            d = CF.synthetic_dataset(kind, n, seed)
            assert np.array_equal(d.features, X) and np.array_equal(d.labels, y) and d.n_classes == ncls
    path = tmp_path / "d.csv"
    path.write_text("x1,name,x2,label\n1.5,a,-2,cat\r\n3,b,4e-1,dog\n\n-0.25,c,7,cat\n")
    text = f"[problem]\nkind = mlp\ncsv_path = {path}\nfeature_cols = x2, x1\nlayers = 2, 4, 2\n"
    want = harness.build_problem(text)
    got = CF.problem_data(CF.parse_config_text(text))
    assert np.array_equal(got.dataset.features, want["X"]) and np.array_equal(got.dataset.labels, want["y"])
    assert got.dataset.n_classes == want["n_classes"] == 2


def fake_result(rows=3):
    return TrainResult(np.zeros(4), np.array([1.5, 0.25, 1e-7][:rows]), np.array([np.nan, 0.5, 1.0][:rows]),
                       np.array([0.1, np.nan, 0.3][:rows]), np.arange(rows), np.array([True, False, True][:rows]),
                       2, 1, np.array([0, 0, 1][:rows]), np.array([0, 1, -1][:rows]), np.array([0.5, 1.25, 2.0][:rows]),
                       1234, {"D_shard": 44, "B": 7, "w": 4}, 12.5)


def test_artifact_writers(tmp_path):
    res = fake_result()
    p = A.RunPaths.in_dir(str(tmp_path))
    A.write_metrics_csv(p.metrics_csv, "dho2", res)
    lines = open(p.metrics_csv).read().splitlines()
    assert lines[0] == "trainer,outer_k,inner_l,epoch,train_loss,train_acc,residual_norm,wallclock_ms,ese_refresh_flag"
    assert lines[1] == "dho2,0,0,0,1.5,,0.10000000000000001,0.5,1"
    assert lines[3] == "dho2,1,,2,9.9999999999999995e-08,1,0.29999999999999999,2,1"
    A.write_memory_csv(p.memory_csv, [res.memory])
    assert open(p.memory_csv).read().splitlines() == ["rank,object,peak_slots", "0,B,7", "0,D_shard,44", "0,w,4"]
    A.write_ledger_csv(p.ledger_csv, [(0, "all_gather", 8, 0, 4, 4)])
    assert open(p.ledger_csv).read().splitlines()[1] == "0,all_gather,8,0,4,4"
    assert res.epochs_to_loss(0.3) == 2 and res.final_accuracy() == 1.0


def test_memory_report_reads_device_summaries(harness, tmp_path):
    """Our summary.json is readable by the reference's memory_report (same keys and bound)."""
    from paper_2505_00982_b200.api import TrainerConfig
    dirs = []
    for g, n, m in ((1, 12, 8), (1, 100, 20)):
        d = tmp_path / f"r{n}"
        d.mkdir()
        s = A.summary_dict(TrainerConfig(k=2, lanczos_m=m), trainer="dho2", workers=g, gpus=g, seed=1,
                           schedule="concurrent", problem_kind="quadratic", n=n, samples=g, loss_target=0.0)
        res = fake_result()
        A._dump(str(d / "summary.json"), A.finish_summary(s, res, [{"D_shard": n * (m + 1)}], 0.0))
        dirs.append(str(d))
    ours = A.memory_report(dirs[:1])
    ref = harness.memory_report(dirs[:1])
    assert ours == ref and "memory accounting: OK" in ours
    assert "MISMATCH" in A.memory_report(dirs)  # D_shard grew between the runs: flagged like the reference
    assert "MISMATCH" in harness.memory_report(dirs)


def test_comm_report_single_gpu(tmp_path):
    from paper_2505_00982_b200.api import TrainerConfig
    s = A.summary_dict(TrainerConfig(k=2, lanczos_m=8), trainer="dho2", workers=1, gpus=1, seed=1,
                       schedule="concurrent", problem_kind="quadratic", n=12, samples=1, loss_target=0.0)
    A._dump(str(tmp_path / "summary.json"), A.finish_summary(s, fake_result(), [{"D_shard": 108}], 0.0))
    A.write_ledger_csv(str(tmp_path / "ledger.csv"), [])
    rep = A.comm_report(str(tmp_path))
    assert "communication ledger: OK" in rep and "(conserved)" in rep
