"""CPU-side checks of the drop-in boundary: libdho2gpu.so loads without a GPU, exports every symbol
include/dho2gpu.h declares, and its host bookkeeping (rng, shards, budget, permutations, sample
and curvature indices, the synthetic dataset) is bit-exact with the CPU checker."""
import os
import re

import numpy as np
import pytest

import paper_2505_00982_b200 as d
from paper_2505_00982_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dho2gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dho2g_[a-z0-9_]+)\s*\(", src)) - {"dho2g_host_hvp"})


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 55
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) == set(_lib.EXPORTED), set(syms) ^ set(_lib.EXPORTED)


def test_no_cpu_fallback_in_product():
    """The product package never imports the checker."""
    pkg = os.path.join(ROOT, "paper_2505_00982_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle.bindings" not in txt and "libdho2oracle" not in txt and "libdho2ref" not in txt, f


def test_rng_bitwise(port):
    for seed in (0, 1, 99, 2**64 - 3):
        assert (d.rng_u64(seed, 300) == port.rng_u64(seed, 300)).all()
        assert (d.rng_normal(seed, 301) == port.rng_normal(seed, 301)).all()
        assert (d.shuffle_iota(seed, 777) == port.shuffle_iota(seed, 777)).all()


def test_shard_and_budget(port):
    for n, C in [(10, 8), (203530, 4), (100989962, 8), (7, 7), (0, 3)]:
        for r in range(C):
            assert d.shard_for_rank(n, C, r) == port.shard(n, C, r)
    for args in [(8, 0, 10000), (1, 1, 100), (3, 2, 10), (10, 0, 203530), (32, 0, 100989962)]:
        assert d.lanczos_budget(*args) == port.lanczos_budget(*args)
    with pytest.raises(d.ArgumentError):
        d.lanczos_budget(6, 5, 10)
    with pytest.raises(d.ArgumentError):
        d.lanczos_budget(0, 0, 10)
    with pytest.raises(d.ArgumentError):
        d.shard_for_rank(10, 0, 0)


def test_permutations_and_indices(port):
    from oracle.bindings import CpuChecker
    assert (d.epoch_permutation(1280, 7, 0) == port.epoch_permutation(1280, 7, 0)).all()
    assert (d.epoch_permutation(5120, 7, 3) == port.epoch_permutation(5120, 7, 3)).all()
    # curvature batch (trainer.cpp:108-114): Rng(mix_seed(seed, 0xc0ffee + refresh)).shuffle(iota)
    for refresh in range(3):
        want = port.shuffle_iota(_mix(1, 0xC0FFEE + refresh), 1280)[:128]
        assert (d.curvature_indices(1280, 128, 1, refresh) == want).all()
    perm = port.epoch_permutation(5120, 7, 1)
    for worker in range(4):
        b, e = port.shard(5120, 4, worker)
        for rnd in (0, 9):
            want = perm[b + (rnd * 128 + np.arange(128)) % (e - b)]
            assert (d.batch_indices(perm, 5120, 4, worker, rnd, 128) == want).all()


def _mix(seed, salt):
    M = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_mix_seed():
    for s, salt in [(1, 0xBEEF), (7, 0xC0FFEE + 3), (2**63, 5)]:
        assert d.mix_seed(s, salt) == _mix(s, salt)


def test_blobs_dataset_matches_checker():
    from oracle.bindings import blobs_dataset as ref_blobs
    X, y = d.blobs_dataset(300, 20, 10, seed=7)
    Xr, yr = ref_blobs(300, 20, 10, seed=7)
    assert (X == Xr).all() and (y == yr).all()
    assert (np.bincount(y.astype(int)) == 30).all()


def test_mlp_init_params_without_gpu_is_refused():
    """Device objects need a CUDA context; without a GPU the call fails loudly (no fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(d.CudaError):
        d.Context(0)
