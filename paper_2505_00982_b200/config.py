"""Experiment configuration front end: the reference's KvConfig grammar and
problem construction, driving the device path.

harness.cpp:29-255 parses a flat ``key = value`` file with ``[sections]`` (``#`` comments; a key
left unconsumed is an ArgumentError naming it) into an ExperimentConfig (harness.hpp:12-41), and
harness.cpp:261-309 turns it into a TrainerConfig and a Problem. This module restates both and
adds one key the reference lacks, ``[lanczos] m`` (explicit iteration count; the C4 north-star
config needs m = 80 < lanczos_budget), so the same config files run on the GPU::

    cfg = load_config("run.ini")
    rc = run_config(ctx, cfg)        # writes metrics.csv / ledger.csv / memory.csv / summary.json
"""
from __future__ import annotations

import ctypes as C
import math
import re
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

import numpy as np

from . import _lib as L
from .api import (ArgumentError, BaseConfig, Context, Dataset, LanczosOptions, MlpOracle, QuadraticOracle,
                  TrainerConfig, _d, check, rng_normal)

lib = L.lib


@dataclass
class ProblemConfig:
    """harness.hpp:12-32 (defaults)."""
    kind: str = "quadratic"
    n: int = 100
    condition: float = 1e4
    rotation_seed: int = 1
    spectrum: str = ""
    dataset: str = "two-gaussians"
    csv_path: str = ""
    label_col: str = "label"
    feature_cols: List[str] = field(default_factory=list)
    samples: int = 400
    dataset_seed: int = 7
    layers: List[int] = field(default_factory=lambda: [2, 16, 2])
    activation: str = "tanh"
    loss: str = "softmax_ce"


@dataclass
class ExperimentConfig:
    """harness.hpp:34-41 (+ lanczos_m)."""
    trainer: str = "dho2"
    workers: int = 1
    seed: int = 1
    schedule: str = "concurrent"
    out_dir: str = "out"
    loss_target: float = 1e-6
    problem: ProblemConfig = field(default_factory=ProblemConfig)
    train: TrainerConfig = field(default_factory=TrainerConfig)


_U64 = re.compile(r"[0-9]+\Z")
# std::from_chars(double) general format: optional '-', digits with optional fraction, optional exponent,
# or inf / nan (no leading '+', no leading/trailing spaces)
_DBL = re.compile(r"-?(?:(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?|inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)\Z",
                  re.IGNORECASE)


def _trim(s: str) -> str:
    return s.strip(" \t")


class KvConfig:
    """Sectioned key-value store with consumption tracking (harness.cpp:38-176)."""

    def __init__(self, text: str, origin: str):
        self.origin = origin
        self.sections: Dict[str, Dict[str, str]] = {}
        self.consumed = set()
        section = ""
        for lineno, line in enumerate(text.split("\n"), 1):
            if "#" in line:
                line = line[: line.index("#")]
            t = _trim(line)
            if not t:
                continue
            if t[0] == "[":
                if t[-1] != "]":
                    raise ArgumentError(f"{origin}:{lineno}: malformed section")
                section = _trim(t[1:-1])
                self.sections.setdefault(section, {})
                continue
            if "=" not in t:
                raise ArgumentError(f"{origin}:{lineno}: expected key = value")
            eq = t.index("=")
            key, value = _trim(t[:eq]), _trim(t[eq + 1:])
            if not key:
                raise ArgumentError(f"{origin}:{lineno}: empty key")
            self.sections.setdefault(section, {})[key] = value

    def fetch(self, section: str, key: str, parse: Callable[[str], object]):
        sec = self.sections.get(section)
        if sec is None or key not in sec:
            return None
        try:
            out = parse(sec[key])
        except ArgumentError as e:
            raise ArgumentError(f"{self.origin}: field '{key}' in [{section}]: {e}") from None
        self.consumed.add(section + "/" + key)
        return (out,)

    def check_consumed(self):
        for section in sorted(self.sections):
            for key in sorted(self.sections[section]):
                if section + "/" + key not in self.consumed:
                    raise ArgumentError(f"{self.origin}: unknown field '{key}' in [{section}]")

    @staticmethod
    def parse_u64(v: str) -> int:
        if not _U64.match(v) or int(v) >= 1 << 64:
            raise ArgumentError(f"'{v}' is not a nonnegative integer")
        return int(v)

    @staticmethod
    def parse_double(v: str) -> float:
        if not _DBL.match(v):
            raise ArgumentError(f"'{v}' is not a number")
        return float(v)

    @staticmethod
    def parse_bool(v: str) -> bool:
        if v in ("true", "1"):
            return True
        if v in ("false", "0"):
            return False
        raise ArgumentError("expected true|false")

    @staticmethod
    def split_list(v: str) -> List[str]:
        parts = v.split(",")
        out = [_trim(p) for p in parts[:-1]]
        last = _trim(parts[-1])
        if last or out:
            out.append(last)
        return out


def _sigma_preset(name: str) -> float:
    """harness.cpp:168-174."""
    presets = {"resnet-101": 5e-4, "vgg-16": 5e-6, "resnet-152": 5e-7}
    if name not in presets:
        raise ArgumentError(f"sigma_preset: expected resnet-101|vgg-16|resnet-152, got '{name}'")
    return presets[name]


_BASE_KINDS = ("sgd", "momentum", "adam", "adamw")


def parse_config_text(text: str, origin: str = "<text>") -> ExperimentConfig:
    """harness.cpp:181-247, plus [lanczos] m (explicit Lanczos iteration count; 0 = lanczos_budget)."""
    kv = KvConfig(text, origin)
    cfg = ExperimentConfig()
    p, t = cfg.problem, cfg.train
    s, u, r, b = str, KvConfig.parse_u64, KvConfig.parse_double, KvConfig.parse_bool

    def get(sec, key, parse, setter):
        got = kv.fetch(sec, key, parse)
        if got is not None:
            setter(got[0])

    def setp(name):
        return lambda v: setattr(p, name, v)

    def sett(name):
        return lambda v: setattr(t, name, v)

    get("experiment", "trainer", s, lambda v: setattr(cfg, "trainer", v))
    # static_cast<int>(uint64): wraps modulo 2^32 (harness.cpp:102-104)
    get("experiment", "workers", u, lambda v: setattr(cfg, "workers", ((v & 0xFFFFFFFF) ^ 0x80000000) - 0x80000000))
    get("experiment", "seed", u, lambda v: setattr(cfg, "seed", v))
    get("experiment", "schedule", s, lambda v: setattr(cfg, "schedule", v))
    get("experiment", "out", s, lambda v: setattr(cfg, "out_dir", v))

    get("problem", "kind", s, setp("kind"))
    get("problem", "n", u, setp("n"))
    get("problem", "condition", r, setp("condition"))
    get("problem", "rotation_seed", u, setp("rotation_seed"))
    get("problem", "spectrum", s, setp("spectrum"))
    get("problem", "dataset", s, setp("dataset"))
    get("problem", "csv_path", s, setp("csv_path"))
    get("problem", "label_col", s, setp("label_col"))
    get("problem", "feature_cols", KvConfig.split_list, setp("feature_cols"))
    get("problem", "samples", u, setp("samples"))
    get("problem", "dataset_seed", u, setp("dataset_seed"))
    get("problem", "layers", lambda v: [u(x) for x in KvConfig.split_list(v)], setp("layers"))
    get("problem", "activation", s, setp("activation"))
    get("problem", "loss", s, setp("loss"))

    base = BaseConfig()
    got = kv.fetch("optimizer", "base", s)
    if got is not None and got[0]:
        if got[0] not in _BASE_KINDS:  # optimizer.cpp:7-14
            raise ArgumentError(f"base optimizer: expected sgd|momentum|adam|adamw, got '{got[0]}'")
        base.kind = got[0]
    for key in ("lr", "weight_decay", "beta1", "beta2", "eps", "momentum"):
        get("optimizer", key, r, lambda v, key=key: setattr(base, key, v))
    t.base = base
    get("optimizer", "k", u, sett("k"))
    get("optimizer", "l", u, sett("l"))
    get("optimizer", "alpha", r, sett("alpha"))
    get("optimizer", "eigval_floor", r, sett("eigval_floor"))
    get("optimizer", "refresh_interval", u, sett("refresh_interval"))
    get("optimizer", "curvature_batch", u, sett("curvature_batch"))

    get("training", "epochs", u, sett("epochs"))
    get("training", "K", u, sett("outer_rounds"))
    get("training", "P", u, sett("inner_epochs"))
    get("training", "sigma", r, sett("sigma"))
    got = kv.fetch("training", "sigma_preset", s)
    if got is not None and got[0]:
        t.sigma = _sigma_preset(got[0])
    get("training", "batch_size", u, sett("batch_size"))
    get("training", "loss_target", r, lambda v: setattr(cfg, "loss_target", v))
    get("training", "sigma_zero_reduction", b, sett("sigma_zero_reduction"))
    get("training", "debug_hash_checks", b, sett("debug_hash_checks"))

    lz = LanczosOptions()
    get("lanczos", "reorth_safeguard", b, lambda v: setattr(lz, "reorth_safeguard", v))
    get("lanczos", "safeguard_ratio", r, lambda v: setattr(lz, "safeguard_ratio", v))
    get("lanczos", "breakdown_rtol", r, lambda v: setattr(lz, "breakdown_rtol", v))
    get("lanczos", "m", u, sett("lanczos_m"))  # device-path extension
    t.lanczos = lz

    get("model", "bandwidth_gbps", r, sett("model_bandwidth_gbps"))
    get("model", "gflops", r, sett("model_gflops"))

    kv.check_consumed()
    if cfg.workers < 1:
        raise ArgumentError(f"{origin}: field 'workers' must be >= 1")
    return cfg


def load_config(path: str) -> ExperimentConfig:
    """harness.cpp:249-255."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ArgumentError(f"config: cannot open '{path}'") from None
    return parse_config_text(text, path)


def build_trainer_config(cfg: ExperimentConfig) -> TrainerConfig:
    """harness.cpp:261-266: kind from [experiment] trainer, seed from [experiment] seed."""
    if cfg.trainer not in ("sgd", "fosi", "dho2"):
        raise ArgumentError(f"trainer: expected sgd|fosi|dho2, got '{cfg.trainer}'")
    t = cfg.train
    return TrainerConfig(**{**t.__dict__, "kind": cfg.trainer, "seed": cfg.seed})


def synthetic_dataset(kind: str, n_samples: int, seed: int) -> Dataset:
    """generate_synthetic_dataset (oracle.cpp:77-127), bit-exact (library host code)."""
    X, y = np.empty(n_samples * 3), np.empty(n_samples)
    dim, ncls = C.c_size_t(), C.c_size_t()
    check(lib.dho2g_synthetic_dataset(kind.encode(), n_samples, seed, _d(X), _d(y), C.byref(dim), C.byref(ncls)))
    return Dataset(X[: n_samples * dim.value].reshape(n_samples, dim.value).copy(), y, ncls.value, seed)


def load_csv_dataset(path: str, feature_cols: List[str], label_col: str) -> Dataset:
    """load_csv_dataset (oracle.cpp:165-213): labels mapped to first-appearance class indices."""
    try:
        f = open(path)
    except OSError:
        raise ArgumentError(f"csv: cannot open '{path}'") from None
    with f:
        lines = f.read().split("\n")
    if not lines or (len(lines) == 1 and not lines[0]):
        raise ArgumentError(f"csv: missing header row in '{path}'")

    def cells(line):
        return [c.replace("\r", "") for c in line.split(",")]

    header = cells(lines[0])

    def col(name):
        if name not in header:
            raise ArgumentError(f"csv: no column named '{name}'")
        return header.index(name)

    li = col(label_col)
    fi = [j for j in range(len(header)) if j != li] if not feature_cols else [col(c) for c in feature_cols]
    if not fi:
        raise ArgumentError("csv: no feature columns selected")
    feats, labels, names = [], [], {}
    for row, line in enumerate(lines[1:], 1):
        if not line or line == "\r":
            continue
        cs = cells(line)
        if len(cs) != len(header):
            raise ArgumentError(f"csv: row {row} has {len(cs)} cells, expected {len(header)}")
        for j in fi:
            if not _DBL.match(cs[j]):
                raise ArgumentError(f"csv: row {row}, column '{header[j]}': '{cs[j]}' is not numeric")
            feats.append(float(cs[j]))
        labels.append(float(names.setdefault(cs[li], len(names))))
    if not labels:
        raise ArgumentError(f"csv: no data rows in '{path}'")
    return Dataset(np.array(feats).reshape(len(labels), len(fi)), np.array(labels), len(names), 0)


@dataclass
class Problem:
    """trainer.hpp:59-63 on the device: the oracle, its dataset and w0."""
    oracle: object
    dataset: Dataset
    w0: np.ndarray
    kind: str


def quadratic_spectrum(p: ProblemConfig) -> np.ndarray:
    """harness.cpp:271-285: explicit comma list (std::stod), else log-spaced 10^(-c/2) .. 10^(c/2)."""
    if p.spectrum:
        out = []
        for item in p.spectrum.split(","):
            m = re.match(r"\s*([-+]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][-+]?[0-9]+)?|[-+]?inf|[-+]?nan)", item,
                         re.IGNORECASE)
            if not m:
                raise ArgumentError("stod")
            out.append(float(m.group(1)))
        return np.array(out)
    if p.n < 2:
        raise ArgumentError("problem: quadratic needs n >= 2")
    half = 0.5 * math.log10(p.condition)
    return np.array([math.pow(10.0, -half + 2.0 * half * (i / (p.n - 1))) for i in range(p.n)])


def init_params(sizes: List[int], seed: int) -> np.ndarray:
    """MlpOracle::init_params (oracle.cpp:386-394) from the layer sizes (host, bit-exact)."""
    sz = (C.c_size_t * len(sizes))(*sizes)
    dim = C.c_size_t()
    check(lib.dho2g_init_params(sz, len(sizes), seed, None, C.byref(dim)))
    w = np.empty(dim.value)
    check(lib.dho2g_init_params(sz, len(sizes), seed, _d(w), C.byref(dim)))
    return w


@dataclass
class ProblemData:
    """The host side of build_problem: the quadratic spectrum or the dataset, and w0."""
    kind: str
    w0: np.ndarray
    dataset: Dataset
    spectrum: Optional[np.ndarray] = None


def problem_data(cfg: ExperimentConfig) -> ProblemData:
    """harness.cpp:267-309 without the device oracle (bit-exact host arithmetic)."""
    p = cfg.problem
    if p.kind == "quadratic":
        spec = quadratic_spectrum(p)
        if len(spec) == 0 or not np.all(np.isfinite(spec)) or np.any(spec == 0):  # oracle.cpp:234-240
            raise ArgumentError("quadratic oracle: spectrum entries must be nonzero and finite" if len(spec)
                                else "quadratic oracle: empty spectrum")
        w0 = rng_normal((cfg.seed * 0x9E3779B97F4A7C15 + 99) & 0xFFFFFFFFFFFFFFFF, len(spec))
        return ProblemData("quadratic", w0, Dataset.dummy(cfg.workers), spec)
    if p.kind == "mlp":
        if p.csv_path:
            data = load_csv_dataset(p.csv_path, p.feature_cols, p.label_col)
        else:
            data = synthetic_dataset(p.dataset, p.samples, p.dataset_seed)
        if len(p.layers) < 3:
            raise ArgumentError("problem: layers needs >= 3 entries")
        if p.layers[0] != data.features.shape[1]:
            raise ArgumentError("problem: layers front != dataset feature_dim")
        for name, ok, msg in (("activation", p.activation in ("tanh", "relu"), "tanh|relu"),
                              ("loss", p.loss in ("mse", "softmax_ce"), "mse|softmax_ce")):
            if not ok:  # oracle.cpp:292-302
                raise ArgumentError(f"{name}: expected {msg}, got '{getattr(p, name)}'")
        return ProblemData("mlp", init_params(list(p.layers), cfg.seed), data)
    raise ArgumentError(f"problem: field 'kind' must be quadratic|mlp, got '{p.kind}'")


def build_problem(ctx: Context, cfg: ExperimentConfig) -> Problem:
    """harness.cpp:267-309 with device oracles."""
    d = problem_data(cfg)
    if d.kind == "quadratic":
        return Problem(QuadraticOracle(ctx, d.spectrum, cfg.problem.rotation_seed), d.dataset, d.w0, d.kind)
    p = cfg.problem
    return Problem(MlpOracle(ctx, list(p.layers), p.activation, p.loss), d.dataset, d.w0, d.kind)


def run_config(ctx: Context, cfg: ExperimentConfig, out_dir: Optional[str] = None) -> int:
    """run_experiment (harness.cpp:364-440) for a parsed config on the device path."""
    from .artifacts import run_experiment
    if cfg.schedule not in ("concurrent", "round_robin", "random"):  # collectives.cpp:22-28
        raise ArgumentError(f"schedule: expected concurrent|round_robin|random, got '{cfg.schedule}'")
    tcfg = build_trainer_config(cfg)
    prob = build_problem(ctx, cfg)
    try:
        return run_experiment(ctx, tcfg, prob.oracle, prob.dataset, prob.w0, out_dir or cfg.out_dir,
                              workers=cfg.workers, seed=cfg.seed, problem_kind=prob.kind,
                              loss_target=cfg.loss_target, schedule=cfg.schedule)
    finally:
        prob.oracle.close()
