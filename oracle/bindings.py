"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

``CpuChecker("port")`` loads oracle/libdho2oracle.so (our plain-C fp64 restatement,
oracle/dho2_oracle.c) and ``CpuChecker("reference")`` loads oracle/_ref/libdho2ref.so
(the unmodified reference library compiled in place, oracle/Makefile). Both expose the
same methods, so every pin test runs the restatement against the reference.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libdho2oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdho2ref.so")

_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_uint64)
_sp = C.POINTER(C.c_size_t)

BASE_KINDS = {"sgd": 0, "momentum": 1, "adam": 2, "adamw": 3}
TRAINERS = {"sgd": 0, "fosi": 1, "dho2": 2}


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Op(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_size_t), ("mat", _dp), ("sizes", _sp), ("n_sizes", C.c_int),
                ("act", C.c_int), ("loss", C.c_int), ("w", _dp), ("X", _dp), ("y", _dp), ("B", C.c_size_t),
                ("ncls", C.c_size_t), ("rot_seed", C.c_uint64), ("rot", _dp)]


class BaseCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("lr", C.c_double), ("weight_decay", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("momentum", C.c_double)]


class TrainCfg(C.Structure):
    _fields_ = [("trainer", C.c_int), ("base", BaseCfg), ("k", C.c_size_t), ("l", C.c_size_t),
                ("alpha", C.c_double), ("eigval_floor", C.c_double), ("refresh_interval", C.c_size_t),
                ("curvature_batch", C.c_size_t), ("reorth_safeguard", C.c_int), ("safeguard_ratio", C.c_double),
                ("breakdown_rtol", C.c_double), ("sigma", C.c_double), ("outer_rounds", C.c_size_t),
                ("inner_epochs", C.c_size_t), ("sigma_zero_reduction", C.c_int), ("epochs", C.c_size_t),
                ("batch_size", C.c_size_t), ("seed", C.c_uint64)]


def base_cfg(kind="adamw", lr=1e-3, weight_decay=0.05, beta1=0.9, beta2=0.999, eps=1e-8, momentum=0.9):
    """BaseConfig defaults of optimizer.hpp:16-24."""
    return BaseCfg(BASE_KINDS[kind], lr, weight_decay, beta1, beta2, eps, momentum)


def train_cfg(trainer="dho2", base=None, k=8, l=0, alpha=0.1, eigval_floor=1e-6, refresh_interval=0,
              curvature_batch=512, reorth_safeguard=True, safeguard_ratio=1e-6, breakdown_rtol=1e-10, sigma=1e-2,
              outer_rounds=25, inner_epochs=4, sigma_zero_reduction=False, epochs=100, batch_size=16, seed=1):
    """TrainerConfig defaults of trainer.hpp:26-57."""
    return TrainCfg(TRAINERS[trainer], base or base_cfg(), k, l, alpha, eigval_floor, refresh_interval,
                    curvature_batch, int(reorth_safeguard), safeguard_ratio, breakdown_rtol, sigma, outer_rounds,
                    inner_epochs, int(sigma_zero_reduction), epochs, batch_size, seed)


class CpuChecker:
    def __init__(self, kind="port"):
        self.kind = kind
        path = REF_SO if kind == "reference" else PORT_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (see __graft_entry__.build)")
        self.lib = C.CDLL(path)
        p = "ref_" if kind == "reference" else "orc_"
        self.p = p
        L = self.lib
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "rng_u64").argtypes = [C.c_uint64, C.c_size_t, _up]
        getattr(L, p + "rng_normal").argtypes = [C.c_uint64, C.c_size_t, _dp]
        getattr(L, p + "rng_uniform").argtypes = [C.c_uint64, C.c_size_t, _dp]
        getattr(L, p + "rng_shuffle_iota").argtypes = [C.c_uint64, C.c_size_t, _up]
        getattr(L, p + "shard").argtypes = [C.c_size_t, C.c_int, C.c_int, _sp, _sp]
        getattr(L, p + "lanczos_budget").argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, _sp]
        getattr(L, p + "seeded_unit_gaussian").argtypes = [C.c_size_t, C.c_uint64, _dp]
        getattr(L, p + "epoch_permutation").argtypes = [C.c_size_t, C.c_uint64, C.c_uint64, _up]
        if kind == "reference":
            L.ref_epoch_permutation.restype = C.c_int
        getattr(L, p + "mlp_dim").argtypes = [_sp, C.c_int, _sp]
        getattr(L, p + "mlp_init").argtypes = [_sp, C.c_int, C.c_uint64, _dp]
        for f in ("value", "grad", "accuracy"):
            getattr(L, p + "mlp_" + f).argtypes = [_sp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_size_t, C.c_size_t, _dp]
        getattr(L, p + "mlp_hvp").argtypes = [_sp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_size_t, C.c_size_t,
                                     _dp]
        getattr(L, p + "tridiag_eig").argtypes = [C.c_size_t, _dp, _dp, _dp, _dp]
        lz = [C.POINTER(Op), C.c_int, C.c_size_t, C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_size_t,
              C.c_size_t, _dp, _dp, _sp, C.POINTER(C.c_int), _sp, _dp, _dp, _dp]
        if kind == "reference":
            lz = lz + [_dp]
        getattr(L, p + "lanczos").argtypes = lz
        getattr(L, p + "base_steps").argtypes = [C.POINTER(BaseCfg), C.c_size_t, C.c_int, _dp, _dp, _dp]
        getattr(L, p + "deltas_seq").argtypes = [C.POINTER(BaseCfg), C.c_size_t, C.c_size_t, _dp, _dp, C.c_int, _dp, _dp,
                                        _dp, C.c_double, C.c_double, C.c_double, C.c_int, _dp, _dp]
        getattr(L, p + "admm_round").argtypes = [C.c_size_t, C.c_double, _dp, _dp, _dp, _dp, _dp]
        tr = [C.POINTER(TrainCfg), _sp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_size_t, C.c_size_t, C.c_uint64,
              _dp, C.c_int, _dp, C.c_size_t, _sp, _dp, _dp, _dp, C.POINTER(C.c_int64), _sp, _sp]
        if kind == "reference":
            tr = tr + [_dp]
            L.ref_set_parallel.argtypes = [C.c_int]
        getattr(L, p + "train_mlp").argtypes = tr
        # QuadraticOracle (oracle.cpp:233-286)
        getattr(L, p + "quadratic_rotation").argtypes = [C.c_size_t, C.c_uint64, _dp]
        self._qapply = "quadratic_apply" if kind == "reference" else "quadratic_apply_seeded"
        getattr(L, p + self._qapply).argtypes = [_dp, C.c_size_t, C.c_uint64, _dp, _dp, _dp]
        tq = [C.POINTER(TrainCfg), _dp, C.c_size_t, C.c_uint64, C.c_size_t, _dp, C.c_int, _dp, C.c_size_t, _sp, _dp,
              _dp, _dp, C.POINTER(C.c_int64), _sp, _sp]
        if kind == "reference":
            tq = tq + [_dp]
        getattr(L, p + "train_quadratic").argtypes = tq

    # -- helpers
    def _call(self, name, *args):
        rc = getattr(self.lib, self.p + name)(*args)
        if rc:
            raise CheckerError(rc, getattr(self.lib, self.p + "last_error")().decode())

    def set_parallel(self, on: bool):
        if self.kind == "reference":
            self.lib.ref_set_parallel(int(on))

    def max_threads(self):
        return self.lib.ref_max_threads() if self.kind == "reference" else 1

    # -- rng / bookkeeping (rng.hpp, collectives.cpp:10-20, oracle.cpp:56-62)
    def rng_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        getattr(self.lib, self.p + "rng_u64")(seed, n, out.ctypes.data_as(_up))
        return out

    def rng_normal(self, seed, n):
        out = np.empty(n)
        getattr(self.lib, self.p + "rng_normal")(seed, n, _d(out))
        return out

    def rng_uniform(self, seed, n):
        out = np.empty(n)
        getattr(self.lib, self.p + "rng_uniform")(seed, n, _d(out))
        return out

    def shuffle_iota(self, seed, n):
        out = np.empty(n, np.uint64)
        getattr(self.lib, self.p + "rng_shuffle_iota")(seed, n, out.ctypes.data_as(_up))
        return out

    def shard(self, n, world, rank):
        b, e = C.c_size_t(), C.c_size_t()
        self._call("shard", n, world, rank, C.byref(b), C.byref(e))
        return b.value, e.value

    def lanczos_budget(self, k, l, n):
        m = C.c_size_t()
        self._call("lanczos_budget", k, l, n, C.byref(m))
        return m.value

    def seeded_unit_gaussian(self, n, seed):
        out = np.empty(n)
        self._call("seeded_unit_gaussian", n, seed, _d(out))
        return out

    def epoch_permutation(self, N, shuffle_seed, epoch):
        out = np.empty(N, np.uint64)
        getattr(self.lib, self.p + "epoch_permutation")(N, shuffle_seed, epoch, out.ctypes.data_as(_up))
        return out

    # -- MLP (oracle.cpp:288-687)
    @staticmethod
    def _sizes(sizes):
        return (C.c_size_t * len(sizes))(*sizes)

    def mlp_dim(self, sizes):
        d = C.c_size_t()
        self._call("mlp_dim", self._sizes(sizes), len(sizes), C.byref(d))
        return d.value

    def mlp_init(self, sizes, seed):
        w = np.empty(self.mlp_dim(sizes))
        self._call("mlp_init", self._sizes(sizes), len(sizes), seed, _d(w))
        return w

    def _mlp(self, f, sizes, act, loss, w, X, y, ncls, out):
        X, y, w = _f64(X), _f64(y), _f64(w)
        self._call("mlp_" + f, self._sizes(sizes), len(sizes), act, loss, _d(w), _d(X), _d(y), len(y), ncls,
                   _d(out))
        return out

    def mlp_value(self, sizes, w, X, y, ncls=10, act=0, loss=0):
        return float(self._mlp("value", sizes, act, loss, w, X, y, ncls, np.empty(1))[0])

    def mlp_accuracy(self, sizes, w, X, y, ncls=10, act=0, loss=0):
        return float(self._mlp("accuracy", sizes, act, loss, w, X, y, ncls, np.empty(1))[0])

    def mlp_grad(self, sizes, w, X, y, ncls=10, act=0, loss=0):
        return self._mlp("grad", sizes, act, loss, w, X, y, ncls, np.empty(len(w)))

    def mlp_hvp(self, sizes, w, v, X, y, ncls=10, act=0, loss=0):
        X, y, w, v = _f64(X), _f64(y), _f64(w), _f64(v)
        out = np.empty(len(w))
        self._call("mlp_hvp", self._sizes(sizes), len(sizes), act, loss, _d(w), _d(v), _d(X), _d(y), len(y), ncls,
                   _d(out))
        return out

    # -- linalg.cpp:140-226
    def tridiag_eig(self, diag, off):
        diag, off = _f64(diag), _f64(off)
        n = len(diag)
        vals, vecs = np.empty(n), np.empty(n * n)
        self._call("tridiag_eig", n, _d(diag), _d(off) if n > 1 else None, _d(vals), _d(vecs))
        return vals, vecs.reshape(n, n).T  # columns are eigenvectors

    # -- dist_lanczos.cpp:31-158
    def lanczos(self, op: dict, m, seed, k=0, l=0, workers=1, safeguard=True, safeguard_ratio=1e-6,
                breakdown_rtol=1e-10, want_basis=True):
        n = op["n"]
        keep = []
        mat = op.get("mat")
        if mat is not None:
            mat = _f64(np.asarray(mat, np.float64).T.reshape(-1) if np.ndim(mat) == 2 else mat)
            keep.append(mat)
        o = Op(op["kind"], n, _d(mat) if mat is not None else None, None, 0, 0, 0, None, None, None, 0, 0, 0, None)
        if op["kind"] == 1 and op.get("rot_seed", 0):
            o.rot_seed = op["rot_seed"]
            if self.kind != "reference":
                Q = self.quadratic_rotation(n, op["rot_seed"])
                Qc = _f64(Q.T.reshape(-1))
                keep.append(Qc)
                o.rot = _d(Qc)
        if op["kind"] == 2:
            sizes = self._sizes(op["sizes"])
            w, X, y = _f64(op["w"]), _f64(op["X"]), _f64(op["y"])
            keep += [sizes, w, X, y]
            o.sizes, o.n_sizes, o.act, o.loss = sizes, len(op["sizes"]), op.get("act", 0), op.get("loss", 0)
            o.w, o.X, o.y, o.B, o.ncls = _d(w), _d(X), _d(y), len(y), op.get("ncls", 10)
        diag, off = np.zeros(m + 1), np.zeros(max(m, 1))
        iters, sg = C.c_size_t(), C.c_size_t()
        bd = C.c_int()
        basis = np.zeros(n * (m + 1)) if want_basis else None
        r = k + l
        ev, evec = np.zeros(max(r, 1)), np.zeros(n * max(r, 1))
        args = [C.byref(o), workers, m, seed, int(safeguard), safeguard_ratio, breakdown_rtol, k, l, _d(diag),
                _d(off), C.byref(iters), C.byref(bd), C.byref(sg), _d(basis), _d(ev), _d(evec)]
        wall = C.c_double()
        if self.kind == "reference":
            args.append(C.byref(wall))
        self._call("lanczos", *args)
        it = iters.value
        keff = min(k, it)
        leff = min(l, it - keff)
        rr = keff + leff
        out = dict(diag=diag[:it].copy(), off=off[:max(it - 1, 0)].copy() if bd.value else off[:it].copy(),
                   iterations=it, breakdown=bool(bd.value), safeguard_passes=sg.value,
                   eigvals=ev[:rr].copy(), eigvecs=evec[:n * rr].reshape(rr, n).T.copy(), wall_ms=wall.value)
        if want_basis:
            cols = it if bd.value else it + 1
            out["basis"] = basis[:n * cols].reshape(cols, n).T.copy()
        return out

    # -- QuadraticOracle, oracle.cpp:233-286
    def quadratic_rotation(self, n, rotation_seed):
        """The rotation Q (n x n) of QuadraticOracle(spectrum, rotation_seed)."""
        Q = np.zeros(n * n)
        self._call("quadratic_rotation", n, rotation_seed, _d(Q))
        return Q.reshape(n, n).T.copy()  # column-major storage -> Q[i, j]

    def quadratic_apply(self, spectrum, rotation_seed, x):
        """(apply_h(x), value(x)) of QuadraticOracle(spectrum, rotation_seed)."""
        spectrum, x = _f64(spectrum), _f64(x)
        out, val = np.empty(len(spectrum)), C.c_double()
        self._call(self._qapply, _d(spectrum), len(spectrum), rotation_seed, _d(x), _d(out), C.byref(val))
        return out, val.value

    # -- optimizer.cpp:37-154
    def base_steps(self, cfg, g_seq, w):
        g_seq, w = _f64(g_seq), _f64(w)
        T, n = g_seq.shape
        out = np.empty((T, n))
        self._call("base_steps", C.byref(cfg), n, T, _d(g_seq), _d(w), _d(out))
        return out

    def deltas_seq(self, cfg, eigvals, V, g_seq, w, alpha, pi=None, sigma=0.0, floor=1e-6, advance=False):
        """fosi_deltas (pi None) / admm_deltas over T steps sharing one BaseOptimizer.
        Returns (newton[T,n], base[T,n], w_after)."""
        g_seq, w = _f64(g_seq), _f64(w).copy()
        T, n = g_seq.shape
        r = len(eigvals)
        ev = _f64(eigvals) if r else np.zeros(1)
        Vc = _f64(np.asarray(V).T.reshape(-1)) if r else np.zeros(1)
        newton, base = np.empty((T, n)), np.empty((T, n))
        self._call("deltas_seq", C.byref(cfg), n, r, _d(ev), _d(Vc), T, _d(g_seq),
                   _d(_f64(pi)) if pi is not None else None, _d(w), alpha, sigma, floor, int(advance), _d(newton),
                   _d(base))
        return newton, base, w

    def admm_round(self, sigma, w_a, pi, w_a_after=None):
        w_a, pi = _f64(w_a), _f64(pi)
        n = len(w_a)
        w = np.empty(n)
        pi_out = np.empty(n) if w_a_after is not None else None
        self._call("admm_round", n, sigma, _d(w_a), _d(pi), _d(w), _d(_f64(w_a_after)) if w_a_after is not None
                   else None, _d(pi_out))
        return w, pi_out

    # -- trainer.cpp:273-298
    def train_mlp(self, cfg, sizes, X, y, w0, workers=1, ncls=10, dataset_seed=7, act=0, loss=0, max_rows=4096):
        X, y, w0 = _f64(X), _f64(y), _f64(w0)
        n = len(w0)
        wf = np.empty(n)
        rl, ra, rr = np.empty(max_rows), np.empty(max_rows), np.empty(max_rows)
        re = np.empty(max_rows, np.int64)
        nrows, refr, sg = C.c_size_t(), C.c_size_t(), C.c_size_t()
        args = [C.byref(cfg), self._sizes(sizes), len(sizes), act, loss, _d(X), _d(y), len(y), ncls, dataset_seed,
                _d(w0), workers, _d(wf), max_rows, C.byref(nrows), _d(rl), _d(ra), _d(rr),
                re.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(refr), C.byref(sg)]
        wall = C.c_double()
        if self.kind == "reference":
            args.append(C.byref(wall))
        self._call("train_mlp", *args)
        k = min(nrows.value, max_rows)
        return dict(w_final=wf, loss=rl[:k].copy(), acc=ra[:k].copy(), resid=rr[:k].copy(), epoch=re[:k].copy(),
                    refreshes=refr.value, safeguard_passes=sg.value, wall_ms=wall.value)


def _train_quadratic(self, cfg, spectrum, rotation_seed, w0, workers=1, n_samples=None, max_rows=4096):
    """train() on Problem{QuadraticOracle(spectrum, rotation_seed), Dataset::dummy(n_samples or workers), w0}
    (tests/test_trainer.cpp:14-21)."""
    spectrum, w0 = _f64(spectrum), _f64(w0)
    n = len(spectrum)
    wf = np.empty(n)
    rl, ra, rr = np.empty(max_rows), np.empty(max_rows), np.empty(max_rows)
    re = np.empty(max_rows, np.int64)
    nrows, refr, sg = C.c_size_t(), C.c_size_t(), C.c_size_t()
    args = [C.byref(cfg), _d(spectrum), n, rotation_seed, n_samples or workers, _d(w0), workers, _d(wf), max_rows,
            C.byref(nrows), _d(rl), _d(ra), _d(rr), re.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(refr),
            C.byref(sg)]
    wall = C.c_double()
    if self.kind == "reference":
        args.append(C.byref(wall))
    self._call("train_quadratic", *args)
    k = min(nrows.value, max_rows)
    return dict(w_final=wf, loss=rl[:k].copy(), acc=ra[:k].copy(), resid=rr[:k].copy(), epoch=re[:k].copy(),
                refreshes=refr.value, safeguard_passes=sg.value, wall_ms=wall.value)


CpuChecker.train_quadratic = _train_quadratic


# ---- harness (harness.cpp), reference library only ----------------------------------------------
def _ref_string(fn, *args):
    need = C.c_size_t()
    buf = C.create_string_buffer(1 << 16)
    rc = fn(*args, buf, len(buf), C.byref(need))
    return rc, buf, need


class RefHarness:
    """parse_config_text / build_problem / generate_synthetic_dataset / run_experiment / reports of
    the unmodified reference (oracle/_ref/libdho2ref.so)."""

    def __init__(self):
        self.lib = C.CDLL(REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_parse_config_json.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t, _sp]
        L.ref_build_problem.argtypes = [C.c_char_p, C.c_size_t, _dp, _sp, C.c_size_t, _dp, _dp, _sp, _sp, _sp]
        L.ref_synthetic_dataset.argtypes = [C.c_char_p, C.c_size_t, C.c_uint64, _dp, _dp, _sp, _sp]
        L.ref_run_experiment_text.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_memory_report.argtypes = [C.POINTER(C.c_char_p), C.c_int, C.c_char_p, C.c_size_t, _sp]
        L.ref_comm_report.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, _sp]

    def _err(self, rc):
        if rc:
            raise CheckerError(rc, self.lib.ref_last_error().decode())

    def parse_config(self, text, origin="<text>"):
        import json
        rc, buf, _ = _ref_string(self.lib.ref_parse_config_json, text.encode(), origin.encode())
        self._err(rc)
        return json.loads(buf.value.decode())

    def build_problem(self, text, max_n=1 << 16, max_samples=1 << 14):
        w0 = np.empty(max_n)
        X, y = np.empty(max_samples * 3), np.empty(max_samples)
        n, ns, dim, ncls = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
        self._err(self.lib.ref_build_problem(text.encode(), max_n, _d(w0), C.byref(n), max_samples, _d(X), _d(y),
                                             C.byref(ns), C.byref(dim), C.byref(ncls)))
        return dict(w0=w0[: n.value].copy(), X=X[: ns.value * dim.value].reshape(ns.value, dim.value).copy(),
                    y=y[: ns.value].copy(), n_classes=ncls.value)

    def synthetic_dataset(self, kind, n_samples, seed):
        X, y = np.empty(n_samples * 3), np.empty(n_samples)
        dim, ncls = C.c_size_t(), C.c_size_t()
        self._err(self.lib.ref_synthetic_dataset(kind.encode(), n_samples, seed, _d(X), _d(y), C.byref(dim),
                                                 C.byref(ncls)))
        return X[: n_samples * dim.value].reshape(n_samples, dim.value).copy(), y, ncls.value

    def run_experiment(self, text):
        rc = C.c_int()
        self._err(self.lib.ref_run_experiment_text(text.encode(), C.byref(rc)))
        return rc.value

    def memory_report(self, dirs):
        arr = (C.c_char_p * len(dirs))(*[d.encode() for d in dirs])
        rc, buf, _ = _ref_string(self.lib.ref_memory_report, arr, len(dirs))
        self._err(rc)
        return buf.value.decode()

    def comm_report(self, d):
        rc, buf, _ = _ref_string(self.lib.ref_comm_report, d.encode())
        self._err(rc)
        return buf.value.decode()


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def blobs_dataset(N, D, n_classes=10, seed=7):
    """Build-defined "blobs-D" synthetic data: y_i = i mod K, class means
    mu_c ~ N(0,1)^D, x_i = mu_{y_i} + N(0,1)^D, all drawn from one SplitMix64/Box-Muller stream
    (the reference Rng, rng.hpp:14-68) seeded with `seed`. Returned as fp64 row-major."""
    chk = CpuChecker("port")
    stream = chk.rng_normal(seed * 0x2545F4914F6CDD1D + 0xB10B5, n_classes * D + N * D)
    mu = stream[: n_classes * D].reshape(n_classes, D)
    y = (np.arange(N) % n_classes).astype(np.float64)
    X = mu[(np.arange(N) % n_classes)] + stream[n_classes * D:].reshape(N, D)
    return X, y
