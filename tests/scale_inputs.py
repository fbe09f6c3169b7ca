"""TEST INFRASTRUCTURE ONLY — seeded inputs for the parity-at-scale tests (tests/test_gpu_parity_scale.py)
and their fixture generator (tests/golden/make_scale_fixtures.py).

Large inputs (the C4 update pass: a 100,989,962 x 32 V_hat) are not drawn from the reference Rng on the host:
they come from a counter hash that gives the same bits in C (oracle/ref_shim.cpp `h24`), numpy and torch
(int64 arithmetic that never overflows: every product is < 2^49), so the GPU test can build them on the
device and the fixture script can build them inside the reference process. Every value is a 24-bit integer
times a power of two, i.e. exactly representable in fp32: the fp32 device path and the fp64 reference see
IDENTICAL inputs.
"""
from __future__ import annotations

import numpy as np

M24 = 0xFFFFFF

# C4: 3072-3584x8-10, n = 100,989,962
C4_SIZES = [3072] + [3584] * 8 + [10]
C3_SIZES = [3072, 2048, 2048, 10]
C2_SIZES = [784, 256, 10]

# the C4 update-pass case (optimizer.cpp:81-129): AdamW, r = 32, two consecutive steps
UPD_R = 32
UPD_T = 2
UPD_ALPHA, UPD_SIGMA, UPD_FLOOR = 0.1, 1e-2, 1e-6
# k = 32 Ritz values spanning both signs, the floor (0, 1e-7, -1e-9) and a value whose floored
# denominator lands on zero (-0.01 + sigma) -> the reference's |den| < floor branch
UPD_EIGVALS = np.array([60.0, 45.0, 30.0, 20.0, 12.0, 8.0, 5.0, 3.0, 2.0, 1.5, 1.0, 0.7, 0.5, 0.3, 0.2, 0.1, 0.05,
                        0.02, 1e-2, 5e-3, 1e-3, 1e-4, 1e-7, 0.0, -1e-9, -1e-3, -0.01, -0.1, -0.5, -1.0, -2.0, -5.0])
# scales (powers of two): V_hat columns ~ 2^-13 (unit-ish norm at n = 1e8), g ~ 2^-6, pi ~ 2^-9, w ~ 2^-3
V_SCALE, G_SCALE, PI_SCALE, W_SCALE = 2.0 ** -13, 2.0 ** -6, 2.0 ** -9, 2.0 ** -3
SALT_V, SALT_G, SALT_PI, SALT_W = 100, 10, 2, 3


def h24_np(idx: np.ndarray, salt: int) -> np.ndarray:
    """24-bit counter hash (int64 in, int64 out in [0, 2^24))."""
    i = idx.astype(np.int64, copy=False)
    x = ((i & M24) * 0x9E3779 + (i >> 24) * 0x7F4A7D + salt * 0x2545F5 + 0x1234) & M24
    x = ((x ^ (x >> 12)) * 0x2C1B3D) & M24
    x = ((x ^ (x >> 11)) * 0x297A2D) & M24
    return x ^ (x >> 13)


def unif_np(idx: np.ndarray, salt: int, scale: float) -> np.ndarray:
    """(h24 - 2^23) 2^-23 * scale in [-scale, scale), fp64 holding an fp32-exact value."""
    return (h24_np(idx, salt) - (1 << 23)).astype(np.float64) * (scale * 2.0 ** -23)


def h24_torch(idx, salt: int):
    x = ((idx & M24) * 0x9E3779 + (idx >> 24) * 0x7F4A7D + salt * 0x2545F5 + 0x1234) & M24
    x = ((x ^ (x >> 12)) * 0x2C1B3D) & M24
    x = ((x ^ (x >> 11)) * 0x297A2D) & M24
    return x ^ (x >> 13)


def unif_torch(idx, salt: int, scale: float, dtype):
    return (h24_torch(idx, salt) - (1 << 23)).to(dtype) * (scale * 2.0 ** -23)


def mlp_dim(sizes) -> int:
    return int(sum(sizes[t + 1] * sizes[t] + sizes[t + 1] for t in range(len(sizes) - 1)))


def sample_indices(n: int, sizes=None, count: int = 1 << 14, seed: int = 12345) -> np.ndarray:
    """Sorted unique parameter indices: `count` hashed positions spread over [0, n) plus, for an MLP,
    every parameter of the last layer (W_last then b_last, oracle.hpp:113-141), where the top Hessian
    directions concentrate."""
    j = np.arange(count, dtype=np.int64)
    u = (h24_np(j, seed).astype(np.uint64) << np.uint64(24)) | h24_np(j, seed + 1).astype(np.uint64)
    idx = (u % np.uint64(n)).astype(np.int64)
    if sizes is not None:
        last = sizes[-1] * sizes[-2] + sizes[-1]
        idx = np.concatenate([idx, np.arange(n - last, n, dtype=np.int64)])
    return np.unique(idx)


def f32(a):
    """Round to fp32 and back: the exact values the device path receives."""
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def blobs_scaled(N: int, D: int, n_classes: int, seed: int, mean_scale: float):
    """Non-degenerate "blobs-D": the SURVEY §8d blobs stream with the class means scaled by `mean_scale`
    (x_i = s mu_{y_i} + N(0,1)), so the classes overlap and the loss stays well above zero over the run."""
    from oracle.bindings import CpuChecker
    chk = CpuChecker("port")
    stream = chk.rng_normal(seed * 0x2545F4914F6CDD1D + 0xB10B5, n_classes * D + N * D)
    mu = stream[: n_classes * D].reshape(n_classes, D) * mean_scale
    y = (np.arange(N) % n_classes).astype(np.float64)
    X = mu[(np.arange(N) % n_classes)] + stream[n_classes * D:].reshape(N, D)
    return X, y
