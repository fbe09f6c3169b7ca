"""Host-side mirror of the reference's optimizer API for the DHO2 curvature-and-update path.

Names, argument meaning and error behaviour follow /root/reference/proj/include/dho2/*.hpp
(cited per class); the arithmetic runs in libdho2gpu.so on the GPU. Host vectors are numpy
float64 like dho2::Vector; column-major matrices (TallMatrix) are numpy arrays of shape
(rows, cols).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib as L

lib = L.lib


# ----------------------------------------------------------------------------- errors.hpp:8-36
class Dho2Error(RuntimeError):
    code = -1


class DimensionError(Dho2Error, ValueError):
    code = 1


class ArgumentError(Dho2Error, ValueError):
    code = 2


class NumericError(Dho2Error):
    code = 3


class DivergenceError(Dho2Error):
    code = 4


class DeadlockError(Dho2Error):
    code = 5


class CudaError(Dho2Error):
    code = 6


class NcclError(Dho2Error):
    code = 7


class TrainingDiverged(NumericError):  # trainer.hpp:22-24
    code = 8


_ERRORS = {c.code: c for c in (DimensionError, ArgumentError, NumericError, DivergenceError, DeadlockError, CudaError,
                               NcclError, TrainingDiverged)}


def check(rc: int) -> None:
    if rc:
        msg = lib.dho2g_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, Dho2Error)(msg)


def _d(a):
    return a.ctypes.data_as(L.dp) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _colmajor(M):
    """(rows, cols) array -> flat column-major fp64 (TallMatrix::data layout, linalg.hpp:27)."""
    return np.ascontiguousarray(np.asarray(M, np.float64).T).reshape(-1)


# ----------------------------------------------------------------------------- bookkeeping
def shard_for_rank(n: int, world: int, rank: int):
    """Shard::for_rank (collectives.cpp:10-20) -> (begin, end)."""
    b, e = C.c_size_t(), C.c_size_t()
    check(lib.dho2g_shard(n, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def lanczos_budget(k: int, l: int, n: int) -> int:
    """lanczos.cpp:10-16."""
    m = C.c_size_t()
    check(lib.dho2g_lanczos_budget(k, l, n, C.byref(m)))
    return m.value


def mix_seed(seed: int, salt: int) -> int:
    return int(lib.dho2g_mix_seed(seed, salt))


def rng_u64(seed: int, n: int):
    out = np.empty(n, np.uint64)
    lib.dho2g_rng_u64(seed, n, out.ctypes.data_as(L.up))
    return out


def rng_normal(seed: int, n: int):
    out = np.empty(n)
    lib.dho2g_rng_normal(seed, n, _d(out))
    return out


def shuffle_iota(seed: int, n: int):
    out = np.empty(n, np.uint64)
    lib.dho2g_shuffle_iota(seed, n, out.ctypes.data_as(L.up))
    return out


def epoch_permutation(N: int, shuffle_seed: int, epoch: int):
    """Dataset::epoch_permutation (oracle.cpp:56-62)."""
    out = np.empty(N, np.uint64)
    lib.dho2g_epoch_permutation(N, shuffle_seed, epoch, out.ctypes.data_as(L.up))
    return out


def curvature_indices(N: int, want: int, seed: int, refresh: int):
    """Curvature batch of TrainerRun::refresh_ese (trainer.cpp:108-114)."""
    out = np.empty(min(want, N), np.uint64)
    lib.dho2g_curvature_indices(N, want, seed, refresh, out.ctypes.data_as(L.up))
    return out


def batch_indices(perm, N: int, workers: int, worker: int, rnd: int, batch: int):
    """Per-worker sample indices of TrainerRun::mean_gradient (trainer.cpp:92-99)."""
    perm = np.ascontiguousarray(perm, np.uint64)
    out = np.empty(batch, np.uint64)
    check(lib.dho2g_batch_indices(perm.ctypes.data_as(L.up), N, workers, worker, rnd, batch,
                                  out.ctypes.data_as(L.up)))
    return out


def blobs_dataset(N: int, D: int, n_classes: int = 10, seed: int = 7):
    """Build-defined "blobs-D" synthetic data: y_i = i mod K, x_i = mu_{y_i} + N(0,1)."""
    X = np.empty((N, D))
    y = np.empty(N)
    lib.dho2g_blobs_dataset(N, D, n_classes, seed, _d(X), _d(y))
    return X, y


# ----------------------------------------------------------------------------- context
class LocalFabric:
    """In-process rendezvous for `world` ranks on one GPU (include/dho2gpu.h: dho2g_local_fabric_create): the
    multi-rank data path of the library without NCCL, each rank a Context driven by its own host thread."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib.dho2g_local_fabric_create(world, C.byref(h)))
        self.h, self.world = h, world

    def close(self):
        if self.h:
            lib.dho2g_local_fabric_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One GPU (rank). The reference's Worker (collectives.hpp:88-117) becomes a NCCL rank."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.dho2g_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self._children = weakref.WeakSet()

    def _adopt(self, obj):
        self._children.add(obj)

    def set_option(self, key: str, value: float):
        check(lib.dho2g_ctx_set_option(self.h, key.encode(), float(value)))

    def stat(self, key: str) -> float:
        v = C.c_double()
        check(lib.dho2g_ctx_get_stat(self.h, key.encode(), C.byref(v)))
        return v.value

    def synchronize(self):
        check(lib.dho2g_synchronize(self.h))

    def mark(self, i: int):
        """Record CUDA event `i` on the library's stream."""
        check(lib.dho2g_timer_mark(self.h, i))

    def elapsed_ms(self, i0: int, i1: int) -> float:
        v = C.c_double()
        check(lib.dho2g_timer_ms(self.h, i0, i1, C.byref(v)))
        return v.value

    def kernel_stats(self):
        """{kernel: (ms, launches, algorithmic work)} from the per-launch event timers."""
        out = {}
        for i in range(int(self.stat("kt_names"))):
            buf = C.create_string_buffer(128)
            check(lib.dho2g_ctx_kernel_name(self.h, i, buf, 128))
            name = buf.value.decode()
            out[name] = (self.stat(f"kt.{name}.ms"), self.stat(f"kt.{name}.count"), self.stat(f"kt.{name}.work"))
        return out

    def comm_init_local(self, fabric: "LocalFabric", rank: int):
        """Join an in-process fabric as `rank` (several ranks on one GPU, one host thread each)."""
        check(lib.dho2g_comm_init_local(self.h, fabric.h, rank))

    def comm_init_host(self, rank: int, world: int, allgather):
        """Host-transport communicator (dho2g_comm_init_host): ranks in separate processes, possibly on the same
        GPU, whose collectives go through `allgather(send: bytes) -> bytes` (every rank's `send`, concatenated in
        rank order), e.g. over a gloo process group."""
        def _cb(user, send, recv, nbytes):
            try:
                out = allgather(C.string_at(send, nbytes))
                if len(out) != nbytes * world:
                    return 1
                C.memmove(recv, out, len(out))
                return 0
            except Exception:  # noqa: BLE001 — reported to the library as a failed collective
                return 1
        self._host_ag = L.HOST_ALLGATHER(_cb)  # kept alive with the context
        check(lib.dho2g_comm_init_host(self.h, rank, world, self._host_ag, None))

    def ledger(self):
        """This rank's communication ledger rows (CommLedger::Row, collectives.hpp:58-65):
        (event, op, floats, rank, sent, received). Empty on a single GPU."""
        rows = []
        ev, fl, se, rc = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        rk = C.c_int()
        op = C.create_string_buffer(32)
        for i in range(int(lib.dho2g_ctx_ledger_rows(self.h))):
            check(lib.dho2g_ctx_ledger_row(self.h, i, C.byref(ev), op, 32, C.byref(fl), C.byref(rk), C.byref(se),
                                           C.byref(rc)))
            rows.append((ev.value, op.value.decode(), fl.value, rk.value, se.value, rc.value))
        return rows

    def memory(self):
        """Peak float slots per named device object (SlotMeter::peak, accounting.hpp:11-27)."""
        out = {}
        name = C.create_string_buffer(64)
        v = C.c_int64()
        for i in range(int(lib.dho2g_ctx_memory_count(self.h))):
            check(lib.dho2g_ctx_memory_entry(self.h, i, name, 64, C.byref(v)))
            out[name.value.decode()] = v.value
        return out

    def allgather_host(self, values):
        """All-gather host doubles across ranks (rank order); every rank must call it."""
        x = _f64(np.atleast_1d(values))
        out = np.empty(x.size * self.world)
        check(lib.dho2g_ctx_allgather_host(self.h, _d(x), x.size, _d(out)))
        return out.reshape(self.world, x.size)

    def reset_accounting(self):
        check(lib.dho2g_ctx_accounting_reset(self.h))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.dho2g_nccl_unique_id(buf))
        return buf.raw

    def comm_init(self, nccl_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        check(lib.dho2g_comm_init(self.h, buf, rank, world))

    @property
    def rank(self):
        r, w = C.c_int(), C.c_int()
        check(lib.dho2g_comm_rank(self.h, C.byref(r), C.byref(w)))
        return r.value

    @property
    def world(self):
        r, w = C.c_int(), C.c_int()
        check(lib.dho2g_comm_rank(self.h, C.byref(r), C.byref(w)))
        return w.value

    def close(self):
        if self.h:
            # device objects hold pointers into this context: release them first, users before owners
            for obj in sorted(list(self._children), key=lambda o: getattr(o, "_close_order", 9)):
                try:
                    obj.close()
                except Exception:
                    pass
            lib.dho2g_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def test_gemm(ctx: "Context", A, B, backend: int = 0):
    """One split (hi, lo) GEMM C = A B^T in the ctx operand format (test hook; backend 0 tcgen05, 1 CUDA-core)."""
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    M, K = A.shape
    N = B.shape[0]
    Cm = np.empty((M, N), np.float32)
    fp = C.POINTER(C.c_float)
    check(lib.dho2g_test_gemm(ctx.h, M, N, K, A.ctypes.data_as(fp), B.ctypes.data_as(fp), Cm.ctypes.data_as(fp),
                              backend))
    return Cm


def test_gemm_seg(ctx: "Context", A0, B0, A1=None, B1=None, backend: int = 0, a_mn: int = 0, b_mn: int = 0):
    """Two-segment GEMM C = A0 B0^T + A1 B1^T with K-major (0) or MN-major (1) operand storage (test hook)."""
    A0 = np.ascontiguousarray(A0, np.float32)
    B0 = np.ascontiguousarray(B0, np.float32)
    M, K0 = A0.shape
    N = B0.shape[0]
    if A1 is None:
        A1 = np.zeros((M, 0), np.float32)
        B1 = np.zeros((N, 0), np.float32)
    A1 = np.ascontiguousarray(A1, np.float32)
    B1 = np.ascontiguousarray(B1, np.float32)
    K1 = A1.shape[1]
    Cm = np.empty((M, N), np.float32)
    fp = C.POINTER(C.c_float)
    one = np.zeros(1, np.float32)
    ptr = lambda x: (x if x.size else one).ctypes.data_as(fp)  # noqa: E731
    check(lib.dho2g_test_gemm_seg(ctx.h, M, N, K0, K1, ptr(A0), ptr(A1), ptr(B0), ptr(B1), Cm.ctypes.data_as(fp),
                                  backend, a_mn, b_mn))
    return Cm


# ----------------------------------------------------------------------------- oracle.hpp
@dataclass
class Batch:
    """oracle.hpp:17-23 (features row-major size x feature_dim)."""
    features: np.ndarray
    labels: np.ndarray
    n_classes: int = 0

    @property
    def size(self):
        return len(self.labels)


ACTIVATIONS = {"tanh": 0, "relu": 1}
LOSSES = {"softmax_ce": 0, "mse": 1}


class MlpOracle:
    """MlpOracle (oracle.hpp:113-141) on the GPU: value / grad / hvp / accuracy over host fp64
    buffers, same flat parameter layout (oracle.cpp:304-324)."""

    def __init__(self, ctx: Context, layer_sizes, activation: str = "tanh", loss: str = "softmax_ce"):
        if activation not in ACTIVATIONS:
            raise ArgumentError(f"activation: expected tanh|relu, got '{activation}'")
        if loss not in LOSSES:
            raise ArgumentError(f"loss: expected mse|softmax_ce, got '{loss}'")
        self.ctx = ctx
        self.layer_sizes = list(layer_sizes)
        sizes = (C.c_size_t * len(self.layer_sizes))(*self.layer_sizes)
        h = C.c_void_p()
        check(lib.dho2g_mlp_create(ctx.h, sizes, len(self.layer_sizes), ACTIVATIONS[activation], LOSSES[loss],
                                   C.byref(h)))
        self.h = h
        ctx._adopt(self)

    _close_order = 6

    def dim(self) -> int:
        return int(lib.dho2g_mlp_dim(self.h))

    def init_params(self, seed: int):
        w = np.empty(self.dim())
        check(lib.dho2g_mlp_init_params(self.h, seed, _d(w)))
        return w

    def _args(self, w, batch: Batch):
        w = _f64(w)
        if w.size != self.dim():
            raise DimensionError("mlp oracle: parameter length mismatch")
        X = _f64(batch.features)
        y = _f64(batch.labels)
        if X.size != y.size * self.layer_sizes[0]:
            raise ArgumentError("mlp oracle: batch feature_dim != input layer size")
        return w, X, y

    def value(self, w, batch: Batch) -> float:
        w, X, y = self._args(w, batch)
        out = C.c_double()
        check(lib.dho2g_mlp_value(self.h, _d(w), _d(X), _d(y), y.size, batch.n_classes, C.byref(out)))
        return out.value

    def grad(self, w, batch: Batch):
        w, X, y = self._args(w, batch)
        g = np.empty(self.dim())
        check(lib.dho2g_mlp_grad(self.h, _d(w), _d(X), _d(y), y.size, batch.n_classes, _d(g)))
        return g

    def hvp(self, w, v, batch: Batch):
        w, X, y = self._args(w, batch)
        v = _f64(v)
        if v.size != self.dim():
            raise DimensionError("mlp oracle: parameter length mismatch")
        hv = np.empty(self.dim())
        check(lib.dho2g_mlp_hvp(self.h, _d(w), _d(v), _d(X), _d(y), y.size, batch.n_classes, _d(hv)))
        return hv

    def accuracy(self, w, batch: Batch) -> Optional[float]:
        w, X, y = self._args(w, batch)
        out = C.c_double()
        check(lib.dho2g_mlp_accuracy(self.h, _d(w), _d(X), _d(y), y.size, batch.n_classes, C.byref(out)))
        return None if out.value < 0 else out.value

    def close(self):
        if self.h:
            lib.dho2g_mlp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- operators (HvpFn)
class Operator:
    _close_order = 4

    def __init__(self, ctx, h, n, keep=()):
        self.ctx, self.h, self.n, self._keep = ctx, h, n, keep
        ctx._adopt(self)

    def close(self):
        if self.h:
            lib.dho2g_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mlp_hvp_operator(ctx: Context, mlp: MlpOracle, w, batch: Batch) -> Operator:
    """The trainer.cpp:116 lambda: v -> mlp.hvp(w, v, curvature_batch), device resident."""
    w, X, y = mlp._args(w, batch)
    h = C.c_void_p()
    check(lib.dho2g_op_mlp(ctx.h, mlp.h, _d(w), _d(X), _d(y), y.size, batch.n_classes, C.byref(h)))
    return Operator(ctx, h, mlp.dim(), keep=(mlp,))


def diagonal_operator(ctx: Context, spectrum) -> Operator:
    """QuadraticOracle(spectrum, 0).apply_h (oracle.cpp:262-268)."""
    s = _f64(spectrum)
    h = C.c_void_p()
    check(lib.dho2g_op_diag(ctx.h, _d(s), s.size, C.byref(h)))
    return Operator(ctx, h, s.size)


class QuadraticOracle:
    """QuadraticOracle (oracle.hpp:84-102, oracle.cpp:233-286) on the device: H = diag(spectrum) for
    rotation_seed 0, else Q^T diag(spectrum) Q with the reference's seeded Gram-Schmidt rotation Q.
    value/grad/hvp ignore the batch, as in the reference. With a communicator, build it after comm_init."""

    _close_order = 4

    def __init__(self, ctx: Context, spectrum, rotation_seed: int = 0):
        s = _f64(spectrum)
        self.ctx, self._spectrum, self.rotation_seed = ctx, s.copy(), int(rotation_seed)
        h = C.c_void_p()
        check(lib.dho2g_op_quadratic(ctx.h, _d(s), s.size, self.rotation_seed, C.byref(h)))
        self.h = h
        self.n = s.size
        ctx._adopt(self)

    def dim(self) -> int:
        return self.n

    def spectrum(self):
        return self._spectrum.copy()

    def rotated(self) -> bool:
        return self.rotation_seed != 0

    def _apply(self, x, want_value):
        x = _f64(x)
        if x.size != self.n:
            raise DimensionError("quadratic oracle: dimension mismatch")
        out = np.empty(self.n)
        v = C.c_double()
        check(lib.dho2g_op_apply(self.h, _d(x), _d(out), C.byref(v) if want_value else None))
        return out, v.value

    def apply_h(self, x):
        return self._apply(x, False)[0]

    def value(self, w, batch=None) -> float:
        return self._apply(w, True)[1]

    def grad(self, w, batch=None):
        return self.apply_h(w)

    def hvp(self, w, v, batch=None):
        return self.apply_h(v)

    def accuracy(self, w, batch=None):
        return None

    def operator(self):
        """The HvpFn view for lanczos_distributed (shares this oracle's device state)."""
        return _BorrowedOperator(self)

    def close(self):
        if self.h:
            lib.dho2g_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _BorrowedOperator:
    def __init__(self, owner):
        self._owner = owner
        self.ctx, self.n = owner.ctx, owner.n

    @property
    def h(self):
        return self._owner.h

    def close(self):
        pass


def quadratic_operator(ctx: Context, spectrum, rotation_seed: int = 0) -> Operator:
    """QuadraticOracle(spectrum, rotation_seed).apply_h as a Lanczos operator (oracle.cpp:262-272)."""
    s = _f64(spectrum)
    h = C.c_void_p()
    check(lib.dho2g_op_quadratic(ctx.h, _d(s), s.size, int(rotation_seed), C.byref(h)))
    return Operator(ctx, h, s.size)


def dense_operator(ctx: Context, H) -> Operator:
    """matrix_hvp of the reference tests (test_support.hpp:74-82)."""
    H = np.asarray(H, np.float64)
    n = H.shape[0]
    flat = _colmajor(H)
    h = C.c_void_p()
    check(lib.dho2g_op_dense(ctx.h, _d(flat), n, C.byref(h)))
    return Operator(ctx, h, n)


def host_operator(ctx: Context, fn: Callable[[np.ndarray], np.ndarray], n: int) -> Operator:
    """Any host HvpFn (lanczos.hpp:11); called once per Lanczos iteration."""

    def tramp(_user, v, out, nn):
        vin = np.ctypeslib.as_array(v, shape=(nn,))
        res = np.asarray(fn(vin.copy()), np.float64)
        np.ctypeslib.as_array(out, shape=(nn,))[:] = res

    cb = L.HOST_HVP(tramp)
    h = C.c_void_p()
    check(lib.dho2g_op_host(ctx.h, cb, None, n, C.byref(h)))
    return Operator(ctx, h, n, keep=(cb,))


# ----------------------------------------------------------------------------- lanczos.hpp / dist_lanczos.hpp
@dataclass
class LanczosOptions:
    """lanczos.hpp:17-26."""
    reorth_safeguard: bool = True
    safeguard_ratio: float = 1e-6
    breakdown_rtol: float = 1e-10


@dataclass
class DistLanczosOptions:
    lanczos: LanczosOptions = field(default_factory=LanczosOptions)
    hash_checks: bool = False


@dataclass
class TridiagMatrix:
    diag: np.ndarray
    offdiag: np.ndarray

    def dim(self):
        return len(self.diag)


class ShardedLanczosResult:
    """dist_lanczos.hpp:21-30: this rank's basis rows stay on the GPU; B is host fp64."""

    _close_order = 3

    def __init__(self, ctx, h, m):
        self.ctx, self.h, self.m = ctx, h, m
        ctx._adopt(self)
        diag, off = np.zeros(m + 1), np.zeros(m + 1)
        it, bd, sg, b, e = C.c_size_t(), C.c_int(), C.c_size_t(), C.c_size_t(), C.c_size_t()
        check(lib.dho2g_lanczos_result(h, _d(diag), _d(off), C.byref(it), C.byref(bd), C.byref(sg), C.byref(b),
                                       C.byref(e)))
        self.iterations = it.value
        self.breakdown = bool(bd.value)
        self.safeguard_passes = sg.value
        self.shard = (b.value, e.value)
        noff = self.iterations - 1 if self.breakdown else self.iterations
        self.tridiag = TridiagMatrix(diag[: self.iterations].copy(), off[:noff].copy())

    @property
    def basis_shard(self):
        cols = self.iterations if self.breakdown else self.iterations + 1
        rows = self.shard[1] - self.shard[0]
        out = np.empty(rows * cols)
        check(lib.dho2g_lanczos_basis(self.h, _d(out)))
        return out.reshape(cols, rows).T

    def close(self):
        if self.h:
            lib.dho2g_lanczos_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lanczos_distributed(ctx: Context, m: int, op: Operator, n: int, seed: int,
                        opts: Optional[DistLanczosOptions] = None) -> ShardedLanczosResult:
    """dist_lanczos.hpp:32-34 (single GPU == lanczos_single, lanczos.hpp:40-41)."""
    if n != op.n:
        raise DimensionError("lanczos_distributed: hvp returned wrong length")
    o = (opts or DistLanczosOptions()).lanczos
    lo = L.LanczosOpts(int(o.reorth_safeguard), o.safeguard_ratio, o.breakdown_rtol)
    h = C.c_void_p()
    ctx.set_option("hash_checks", int(bool((opts or DistLanczosOptions()).hash_checks)))
    try:
        check(lib.dho2g_lanczos_run(ctx.h, op.h, m, seed, C.byref(lo), C.byref(h)))
    finally:
        ctx.set_option("hash_checks", 0)
    return ShardedLanczosResult(ctx, h, m)


class EseResult:
    """lanczos.hpp:45-52: k largest (descending) then l smallest (ascending) Ritz pairs; the
    eigenvectors are this rank's rows (all rows at world == 1)."""

    _close_order = 2

    def __init__(self, ctx, h, k=0, l=0):
        self.ctx, self.h, self.k, self.l = ctx, h, k, l
        ctx._adopt(self)

    def count(self) -> int:
        return int(lib.dho2g_ese_count(self.h)) if self.h else 0

    @property
    def eigvals(self):
        r = self.count()
        out = np.empty(r)
        if r:
            check(lib.dho2g_ese_eigvals(self.h, _d(out)))
        return out

    def eigvecs_shard(self, rows: int):
        r = self.count()
        out = np.empty(rows * r)
        if r:
            check(lib.dho2g_ese_eigvecs(self.h, _d(out)))
        return out.reshape(r, rows).T

    def eigvecs_full(self, n: int):
        """The full V_hat (n x r) on every rank (extract_ese_distributed's gather_rows,
        dist_lanczos.cpp:148-156); collective at world > 1."""
        r = self.count()
        out = np.empty(n * r)
        if r:
            check(lib.dho2g_ese_gather(self.h, _d(out)))
        return out.reshape(r, n).T

    def eigvecs_to_device(self, ptr: int, ld: int):
        """This rank's V_hat rows (signs applied) into a device fp32 buffer (column-major, leading dimension
        ld), e.g. a torch tensor's data_ptr()."""
        check(lib.dho2g_ese_eigvecs_device(self.h, C.c_void_p(ptr), ld))

    @classmethod
    def from_host(cls, ctx: Context, eigvals, V):
        eigvals = _f64(eigvals)
        V = np.asarray(V, np.float64)
        n, r = V.shape
        h = C.c_void_p()
        check(lib.dho2g_ese_from_host(ctx.h, _d(eigvals), _d(_colmajor(V)), n, r, C.byref(h)))
        return cls(ctx, h, r, 0)

    @classmethod
    def from_device(cls, ctx: Context, eigvals, V_ptr: int, ld: int, n: int, r: int):
        """From a device-resident fp32 V (column-major, leading dimension ld, e.g. a torch tensor's
        data_ptr()); copied device to device."""
        eigvals = _f64(eigvals)
        h = C.c_void_p()
        check(lib.dho2g_ese_from_device(ctx.h, _d(eigvals), C.c_void_p(V_ptr), ld, n, r, C.byref(h)))
        return cls(ctx, h, r, 0)

    def close(self):
        if self.h:
            lib.dho2g_ese_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def extract_ese_distributed(ctx: Context, state: ShardedLanczosResult, k: int, l: int,
                            hash_check: bool = False) -> EseResult:
    """dist_lanczos.hpp:39-41: device tql2 + selection + Ritz vectors (V_hat stays sharded); hash_check: B
    compared across ranks first (DivergenceError "B differs across ranks")."""
    h = C.c_void_p()
    ctx.set_option("hash_checks", int(bool(hash_check)))
    try:
        check(lib.dho2g_extract_ese(ctx.h, state.h, k, l, C.byref(h)))
    finally:
        ctx.set_option("hash_checks", 0)
    return EseResult(ctx, h, k, l)


def select_extreme_indices(count: int, k: int, l: int):
    """lanczos.cpp:72-80."""
    return [count - 1 - j for j in range(k)] + list(range(l))


# ----------------------------------------------------------------------------- optimizer.hpp
BASE_KINDS = {"sgd": 0, "momentum": 1, "adam": 2, "adamw": 3}


@dataclass
class BaseConfig:
    """optimizer.hpp:16-24."""
    kind: str = "adamw"
    lr: float = 1e-3
    weight_decay: float = 0.05
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    momentum: float = 0.9

    def to_c(self):
        if self.kind not in BASE_KINDS:
            raise ArgumentError(f"base optimizer: expected sgd|momentum|adam|adamw, got '{self.kind}'")
        return L.BaseCfg(BASE_KINDS[self.kind], self.lr, self.weight_decay, self.beta1, self.beta2, self.eps,
                         self.momentum)


class BaseOptimizer:
    """optimizer.hpp:28-46 with device-resident moments."""

    def __init__(self, ctx: Context, cfg: BaseConfig, n: int):
        self.ctx, self.cfg, self.n = ctx, cfg, n
        h = C.c_void_p()
        c = cfg.to_c()
        check(lib.dho2g_opt_create(ctx.h, C.byref(c), n, C.byref(h)))
        self.h = h
        ctx._adopt(self)

    _close_order = 5

    def step(self, g, w):
        g, w = _f64(g), _f64(w)
        if g.size != self.n:
            raise DimensionError("BaseOptimizer: gradient length mismatch")
        d = np.empty(self.n)
        check(lib.dho2g_opt_step(self.h, _d(g), _d(w), _d(d)))
        return d

    def close(self):
        if self.h:
            lib.dho2g_opt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Deltas:
    newton: np.ndarray
    base: np.ndarray


def _deltas(g, pi, ese: Optional[EseResult], base: BaseOptimizer, w, alpha, sigma, floor):
    g, w = _f64(g), _f64(w)
    n = g.size
    if pi is not None:
        pi = _f64(pi)
        if pi.size != n:
            raise DimensionError("deltas: pi length mismatch")
    newton, b = np.empty(n), np.empty(n)
    check(lib.dho2g_deltas(base.h, ese.h if (ese is not None and ese.count() > 0) else None, _d(g), _d(pi), _d(w),
                           alpha, sigma, floor, _d(newton), _d(b)))
    return Deltas(newton, b)


def fosi_deltas(g, ese, base: BaseOptimizer, w, alpha, eigval_floor=1e-6) -> Deltas:
    """optimizer.hpp:56-57."""
    return _deltas(g, None, ese, base, w, alpha, 0.0, eigval_floor)


def admm_deltas(g, pi, ese, base: BaseOptimizer, w, alpha, sigma, eigval_floor=1e-6) -> Deltas:
    """optimizer.hpp:62-63."""
    return _deltas(g, pi, ese, base, w, alpha, sigma, eigval_floor)


@dataclass
class AdmmState:
    """optimizer.hpp:66-72."""
    w: np.ndarray
    w_a: np.ndarray
    pi: np.ndarray
    sigma: float
    outer: int = 0


def make_admm_state(w0, sigma: float) -> AdmmState:
    if sigma <= 0.0:
        raise ArgumentError("AdmmState: sigma must be positive")
    w0 = _f64(w0).copy()
    return AdmmState(w0.copy(), w0, np.zeros_like(w0), sigma)


def admm_w_update(ctx: Context, st: AdmmState):
    """w <- w_a + pi / sigma (optimizer.cpp:141-147)."""
    out = np.empty_like(st.w_a)
    check(lib.dho2g_admm_w_update(ctx.h, st.w_a.size, st.sigma, _d(_f64(st.w_a)), _d(_f64(st.pi)), _d(out)))
    st.w = out
    return st.w


def admm_dual_update(ctx: Context, st: AdmmState):
    """pi <- pi + sigma (w_a - w) (optimizer.cpp:149-154)."""
    pi = _f64(st.pi).copy()
    check(lib.dho2g_admm_dual_update(ctx.h, pi.size, st.sigma, _d(_f64(st.w_a)), _d(_f64(st.w)), _d(pi)))
    st.pi = pi
    st.outer += 1


# ----------------------------------------------------------------------------- trainer.hpp
TRAINERS = {"sgd": 0, "fosi": 1, "dho2": 2}


@dataclass
class TrainerConfig:
    """trainer.hpp:26-57 (+ lanczos_m: explicit iteration count)."""
    kind: str = "dho2"
    base: BaseConfig = field(default_factory=BaseConfig)
    k: int = 8
    l: int = 0
    alpha: float = 0.1
    eigval_floor: float = 1e-6
    refresh_interval: int = 0
    curvature_batch: int = 512
    lanczos: LanczosOptions = field(default_factory=LanczosOptions)
    sigma: float = 1e-2
    outer_rounds: int = 25
    inner_epochs: int = 4
    sigma_zero_reduction: bool = False
    epochs: int = 100
    batch_size: int = 16
    seed: int = 1
    lanczos_m: int = 0
    debug_hash_checks: bool = False  # cross-rank B / parameter-replica hashes (trainer.cpp:120-157; context option)
    model_bandwidth_gbps: float = 50.0
    model_gflops: float = 10.0

    def to_c(self):
        if self.kind not in TRAINERS:
            raise ArgumentError(f"trainer: expected sgd|fosi|dho2, got '{self.kind}'")
        return L.TrainCfg(TRAINERS[self.kind], self.base.to_c(), self.k, self.l, self.alpha, self.eigval_floor,
                          self.refresh_interval, self.curvature_batch, int(self.lanczos.reorth_safeguard),
                          self.lanczos.safeguard_ratio, self.lanczos.breakdown_rtol, self.sigma, self.outer_rounds,
                          self.inner_epochs, int(self.sigma_zero_reduction), self.epochs, self.batch_size, self.seed,
                          self.lanczos_m, self.model_bandwidth_gbps, self.model_gflops, int(self.debug_hash_checks))


@dataclass
class Dataset:
    """oracle.hpp:25-54 (features row-major N x D)."""
    features: np.ndarray
    labels: np.ndarray
    n_classes: int
    shuffle_seed: int

    def size(self):
        return len(self.labels)

    @staticmethod
    def dummy(n_samples: int) -> "Dataset":
        """Dataset::dummy (oracle.cpp:64-68): one zero feature, no classes, shuffle seed 0."""
        if n_samples == 0:
            raise ArgumentError("Dataset::dummy: need at least one sample")
        return Dataset(np.zeros((n_samples, 1)), np.zeros(n_samples), 0, 0)


@dataclass
class TrainResult:
    """trainer.hpp:79-89."""
    w_final: np.ndarray
    loss: np.ndarray
    acc: np.ndarray
    residual_norm: np.ndarray
    epoch: np.ndarray
    ese_refresh: np.ndarray
    ese_refreshes: int
    safeguard_passes: int
    outer_k: np.ndarray = None
    inner_l: np.ndarray = None
    wallclock_ms: np.ndarray = None  # modeled clock (trainer.cpp:137-148)
    gs_flops: int = 0
    memory: dict = None  # this rank's SlotMeter (per-rank list in the reference)
    raw_wallclock_ms: float = 0.0

    def final_loss(self):
        return float(self.loss[-1]) if len(self.loss) else 0.0

    def final_accuracy(self):
        """trainer.cpp:27-30: None when the oracle has no accuracy."""
        if not len(self.acc) or np.isnan(self.acc[-1]):
            return None
        return float(self.acc[-1])

    def epochs_to_loss(self, target):
        """trainer.cpp:32-37: epochs run until the first row whose loss is <= target."""
        for e, v in zip(self.epoch, self.loss):
            if v <= target:
                return int(e) + 1
        return None


class Trainer:
    """TrainerRun (trainer.cpp:51-269) on the GPU. step() advances DHO2 steps (inner rounds)."""

    def __init__(self, ctx: Context, cfg: TrainerConfig, mlp, data: Dataset, w0, workers: int = 1,
                 host_resident: bool = False):
        """`mlp` is the Problem's oracle: an MlpOracle, or a QuadraticOracle (then `data` is
        Dataset.dummy(k) as in test_trainer.cpp:14-21; its features are never read)."""
        self.ctx, self.cfg, self.mlp = ctx, cfg, mlp
        X = _f64(data.features)
        y = _f64(data.labels)
        w0 = _f64(w0)
        if w0.size != mlp.dim():
            raise DimensionError("train: w0 length != oracle dimension")
        c = cfg.to_c()
        h = C.c_void_p()
        if isinstance(mlp, QuadraticOracle):
            check(lib.dho2g_trainer_create_quadratic(ctx.h, C.byref(c), mlp.h, y.size, _d(w0), workers, C.byref(h)))
        else:
            check(lib.dho2g_trainer_create(ctx.h, C.byref(c), mlp.h, _d(X), _d(y), y.size, data.n_classes,
                                           data.shuffle_seed, _d(w0), workers, int(host_resident), C.byref(h)))
        self.h = h
        self.n = mlp.dim()
        ctx._adopt(self)

    _close_order = 1

    def step(self, steps: int = 1, with_eval: bool = False):
        check(lib.dho2g_trainer_step(self.h, steps, int(with_eval)))

    def run(self):
        check(lib.dho2g_trainer_run(self.h))

    def params(self):
        w = np.empty(self.n)
        check(lib.dho2g_trainer_params(self.h, _d(w)))
        return w

    def last_loss(self):
        v = C.c_double()
        check(lib.dho2g_trainer_last_loss(self.h, C.byref(v)))
        return v.value

    def stat(self, key: str) -> float:
        v = C.c_double()
        check(lib.dho2g_trainer_stat(self.h, key.encode(), C.byref(v)))
        return v.value

    def eigvals(self):
        buf = np.empty(1024)
        cnt = C.c_size_t()
        check(lib.dho2g_trainer_eigvals(self.h, _d(buf), C.byref(cnt)))
        return buf[: cnt.value].copy()

    def metrics(self):
        n = int(lib.dho2g_trainer_rows(self.h))
        loss, acc, res = np.empty(n), np.empty(n), np.empty(n)
        ep = np.empty(n, np.int64)
        rf = np.empty(n, np.int32)
        check(lib.dho2g_trainer_metrics(self.h, n, _d(loss), _d(acc), _d(res), ep.ctypes.data_as(L.i64p),
                                        rf.ctypes.data_as(L.ip)))
        return loss, acc, res, ep, rf

    def result(self) -> TrainResult:
        loss, acc, res, ep, rf = self.metrics()
        n = len(loss)
        outer, inner = np.empty(n, np.int64), np.empty(n, np.int64)
        wall = np.empty(n)
        check(lib.dho2g_trainer_metrics_ex(self.h, n, outer.ctypes.data_as(L.i64p), inner.ctypes.data_as(L.i64p),
                                           _d(wall)))
        return TrainResult(self.params(), loss, acc, res, ep, rf.astype(bool), int(self.stat("refreshes")),
                           int(self.stat("safeguard_passes")), outer, inner, wall, int(self.stat("gs_flops")),
                           self.ctx.memory())

    def close(self):
        if self.h:
            lib.dho2g_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def train(ctx: Context, cfg: TrainerConfig, mlp: MlpOracle, data: Dataset, w0, workers: int = 1) -> TrainResult:
    """train() (trainer.hpp:95-96 / trainer.cpp:273-298)."""
    import time
    tr = Trainer(ctx, cfg, mlp, data, w0, workers)
    try:
        t0 = time.perf_counter()
        tr.run()
        res = tr.result()
        res.raw_wallclock_ms = (time.perf_counter() - t0) * 1e3  # measured (trainer.cpp:280-296)
        return res
    finally:
        tr.close()
