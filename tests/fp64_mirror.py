"""TEST INFRASTRUCTURE ONLY — an fp64 torch restatement of the reference's hot path, used to compare the
fp32 / split-BF16x3 device path with fp64 arithmetic on FULL vectors at the benchmarked sizes (C3, C4),
where the CPU reference takes minutes to hours per call.

It is not trusted on its own: tests/test_gpu_parity_scale.py first pins it to the UNMODIFIED reference's
outputs stored in tests/golden/scale_*.npz (sampled entries, norms, eigenvalues, B — made by
tests/golden/make_scale_fixtures.py from oracle/_ref), and tests/test_oracle_pin.py pins it to the
compiled reference at small sizes on the CPU. Every function cites the reference lines it restates.
Never imported by the product package.
"""
from __future__ import annotations

import numpy as np
import torch

F64 = torch.float64


class MlpMirror:
    """MlpOracle (oracle.hpp:113-141, oracle.cpp:304-687) in batched fp64 torch. Flat layout per layer:
    W (out x in, row-major) then b (out)."""

    def __init__(self, sizes, device, activation="tanh", loss="softmax_ce"):
        self.sizes = list(sizes)
        self.dev = device
        self.tanh = activation == "tanh"
        self.ce = loss == "softmax_ce"
        self.offs = []
        o = 0
        for t in range(len(sizes) - 1):
            i, u = sizes[t], sizes[t + 1]
            self.offs.append((o, o + u * i, i, u))
            o += u * i + u
        self.n = o

    def layers(self, w):
        return [(w[a:b].view(u, i), w[b:b + u]) for a, b, i, u in self.offs]

    def _act(self, z):
        return torch.tanh(z) if self.tanh else torch.clamp_min(z, 0.0)

    def _act_prime(self, a):  # oracle.cpp:368-370 (evaluated on the activation)
        return 1.0 - a * a if self.tanh else (a > 0).to(F64)

    def forward(self, w, X):
        a = [X]
        L = self.layers(w)
        for t, (W, b) in enumerate(L):
            z = a[-1] @ W.T + b
            a.append(z if t + 1 == len(L) else self._act(z))
        return a

    def _targets(self, y, out):
        if self.ce:
            return None
        T = torch.zeros_like(out)
        if out.shape[1] > 1:
            T[torch.arange(len(y), device=self.dev), y.long()] = 1.0
        else:
            T[:, 0] = y
        return T

    def value(self, w, X, y):  # oracle.cpp:400-449
        out = self.forward(w, X)[-1]
        if self.ce:
            return float((torch.logsumexp(out, 1) - out[torch.arange(len(y), device=self.dev), y.long()]).mean())
        return float((0.5 * ((out - self._targets(y, out)) ** 2).sum(1)).mean())

    def accuracy(self, w, X, y):  # oracle.cpp:649-685 (first maximum on ties)
        out = self.forward(w, X)[-1]
        return float((out.argmax(1) == y.long()).to(F64).mean())

    def _out_delta(self, out, y):
        B = out.shape[0]
        if self.ce:  # oracle.cpp:470-480
            p = torch.softmax(out, 1)
            d = p.clone()
            d[torch.arange(B, device=self.dev), y.long()] -= 1.0
            return d / B, p
        return (out - self._targets(y, out)) / B, None

    def grad(self, w, X, y):  # oracle.cpp:451-522
        a = self.forward(w, X)
        L = self.layers(w)
        d, _ = self._out_delta(a[-1], y)
        g = torch.empty(self.n, dtype=F64, device=self.dev)
        for t in range(len(L) - 1, -1, -1):
            W, _ = L[t]
            o0, o1, i, u = self.offs[t]
            g[o0:o1] = (d.T @ a[t]).reshape(-1)
            g[o1:o1 + u] = d.sum(0)
            if t > 0:
                d = (d @ W) * self._act_prime(a[t])
        return g

    def prepare(self, w, X, y):
        """Caches the v-independent forward state of one (w, batch) point (the HVP operator of a refresh,
        trainer.cpp:116)."""
        self._w, self._y = w, y
        self._a = self.forward(w, X)
        self._d, self._p = self._out_delta(self._a[-1], y)

    def hvp_prepared(self, v):  # oracle.cpp:524-647 (exact Pearlmutter R-op)
        a, L, V = self._a, self.layers(self._w), self.layers(v)
        B = a[0].shape[0]
        ra = [torch.zeros_like(a[0])]
        for t, ((W, _), (VW, vb)) in enumerate(zip(L, V)):
            rz = a[t] @ VW.T + ra[t] @ W.T + vb
            ra.append(rz if t + 1 == len(L) else self._act_prime(a[t + 1]) * rz)
        d = self._d
        if self.ce:  # oracle.cpp:572-587
            p = self._p
            rd = p * (ra[-1] - (p * ra[-1]).sum(1, keepdim=True)) / B
        else:  # oracle.cpp:588-599
            rd = ra[-1] / B
        hv = torch.empty(self.n, dtype=F64, device=self.dev)
        for t in range(len(L) - 1, -1, -1):
            W, _ = L[t]
            VW, _ = V[t]
            o0, o1, i, u = self.offs[t]
            hv[o0:o1] = (rd.T @ a[t] + d.T @ ra[t]).reshape(-1)
            hv[o1:o1 + u] = rd.sum(0)
            if t > 0:
                u_ = d @ W
                ru = d @ VW + rd @ W
                ap = self._act_prime(a[t])
                rap = -2.0 * a[t] * ra[t] if self.tanh else torch.zeros_like(ap)  # :629-635 (0 where ap == 0)
                if self.tanh:
                    rap = torch.where(ap != 0.0, rap, torch.zeros_like(rap))
                d, rd = u_ * ap, ru * ap + u_ * rap
        return hv

    def hvp(self, w, v, X, y):
        self.prepare(w, X, y)
        return self.hvp_prepared(v)


def seeded_unit_gaussian(chk, n, seed, device):
    """lanczos.cpp:18-26: Rng(seed * 0x9e3779b97f4a7c15 + 0x1234567).fill_normal, normalised."""
    s = (seed * 0x9E3779B97F4A7C15 + 0x1234567) % (1 << 64)
    v = torch.tensor(chk.rng_normal(s, n), dtype=F64, device=device)
    return v / torch.linalg.vector_norm(v)


def lanczos(chk, hvp, n, m, seed, device, safeguard=True, safeguard_ratio=1e-6, breakdown_rtol=1e-10):
    """dist_lanczos.cpp:31-119 at one rank (== lanczos.cpp:28-70): classical Gram-Schmidt of the raw h
    against the whole basis, one safeguard pass, breakdown truncation."""
    D = torch.zeros((m + 1, n), dtype=F64, device=device)  # row j = basis column j
    D[0] = seeded_unit_gaussian(chk, n, seed, device)
    diag, off = np.zeros(m + 1), np.zeros(m)
    sg = 0
    for i in range(m):
        v = D[i]
        h = hvp(v)
        if not bool(torch.isfinite(h).all()):
            raise FloatingPointError("lanczos_distributed: hvp returned non-finite values")
        diag[i] = float(h @ v)
        pre = float(torch.linalg.vector_norm(h))
        act = D[: i + 1]

        def project(h):
            return h - act.T @ (act @ h)

        h = project(h)
        beta = float(torch.linalg.vector_norm(h))
        if safeguard and breakdown_rtol * pre < beta < safeguard_ratio * pre:
            h = project(h)
            beta = float(torch.linalg.vector_norm(h))
            sg += 1
        if beta <= breakdown_rtol * pre:
            return dict(D=D[: i + 1], diag=diag[: i + 1], off=off[:i], iterations=i + 1, breakdown=True,
                        safeguard_passes=sg)
        off[i] = beta
        D[i + 1] = h / beta
    return dict(D=D, diag=diag[:m], off=off, iterations=m, breakdown=False, safeguard_passes=sg)


def extract_ese(chk, lz, k, l):
    """dist_lanczos.cpp:121-158 / lanczos.cpp:96-120: tql2 (the reference's, via the pinned checker),
    k largest descending + l smallest ascending, V_hat = D U_sel, sign of the largest-|x| entry (lowest
    index on ties) made positive. Returns (eigvals, V_hat as r x n rows)."""
    me = lz["iterations"]
    vals, vecs = chk.tridiag_eig(lz["diag"][:me], lz["off"][: me - 1])
    idx = [me - 1 - j for j in range(k)] + list(range(l))
    U = torch.tensor(vecs[:, idx], dtype=F64, device=lz["D"].device)
    V = U.T @ lz["D"][:me]
    am = torch.argmax(V.abs(), dim=1)
    sgn = torch.sign(V[torch.arange(V.shape[0], device=V.device), am])
    V = V * torch.where(sgn < 0, -1.0, 1.0).to(F64)[:, None]
    return np.asarray(vals)[idx], V


class BaseOptimizerMirror:
    """BaseOptimizer::step (optimizer.cpp:37-71)."""

    def __init__(self, kind, n, device, lr=1e-3, weight_decay=0.05, beta1=0.9, beta2=0.999, eps=1e-8, momentum=0.9):
        self.kind, self.lr, self.wd, self.b1, self.b2, self.eps, self.mu = kind, lr, weight_decay, beta1, beta2, eps, momentum
        self.t = 0
        self.m = torch.zeros(n, dtype=F64, device=device) if kind != "sgd" else None
        self.v = torch.zeros(n, dtype=F64, device=device) if kind in ("adam", "adamw") else None

    def step(self, g, w):
        self.t += 1
        if self.kind == "sgd":
            return -self.lr * g
        if self.kind == "momentum":
            self.m.mul_(self.mu).add_(g)
            return -self.lr * self.m
        bc1 = 1.0 - self.b1 ** self.t
        bc2 = 1.0 - self.b2 ** self.t
        # magnitude of the terms each element of the step sums (the forward-error scale of evaluating it
        # in fp32 with fp32-stored moments): m = b1 m' + (1 - b1) g can cancel
        mterms = self.b1 * self.m.abs() + (1.0 - self.b1) * g.abs()
        self.m.mul_(self.b1).add_((1.0 - self.b1) * g)
        self.v.mul_(self.b2).add_((1.0 - self.b2) * g * g)
        den = torch.sqrt(self.v / bc2) + self.eps
        d = -self.lr * (self.m / bc1) / den
        self.term_scale = self.lr * (mterms / bc1) / den
        if self.kind == "adamw":
            d = d - self.lr * self.wd * w
            self.term_scale = self.term_scale + self.lr * self.wd * w.abs()
        return d


def floored_eigval(a, floor):  # optimizer.cpp:75-79
    if a == 0.0:
        return floor
    mag = max(abs(a), floor)
    return -mag if a < 0.0 else mag


def split_deltas(g, pi, eigvals, V, base: BaseOptimizerMirror, w, alpha, sigma, floor):
    """optimizer.cpp:81-117. V is r x n (rows = eigenvectors). Returns (newton, base, c, coef, sc)."""
    gt = g if pi is None else g + pi
    c = V @ gt
    coef = torch.empty_like(c)
    for j, a in enumerate(eigvals):
        den = floored_eigval(float(a), floor) + sigma
        if abs(den) < floor:
            den = -floor if den < 0.0 else floor
        coef[j] = c[j] / den
    newton = -alpha * (V.T @ coef)
    g2 = gt - V.T @ c
    s = base.step(g2, w)
    sc = V @ s
    return newton, s - V.T @ sc, c, coef, sc
