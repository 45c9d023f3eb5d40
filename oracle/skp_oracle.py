"""numpy/scipy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Restates, function by function, what ``skpower`` computes on the path
sketch -> power iteration -> orthonormalisation -> small SVD / Nystrom core
(/root/reference/pkg/src/skpower).  The arithmetic is numpy 2.3.5 / scipy
1.18.1 / OpenBLAS 0.3.30 (the versions in this image); the reference only pins
``numpy>=1.24, scipy>=1.10`` (pkg/pyproject.toml:10-13).

This module is the parity checker and the CPU baseline.  It must never be
imported by the product package ``paper_2605_09755_b200``.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

_M64 = (1 << 64) - 1
_HERE = os.path.dirname(os.path.abspath(__file__))


# --------------------------------------------------------------------------
# seeds (sketching.py:46-58)
# --------------------------------------------------------------------------

def substream(seed: int, *idx: int) -> int:
    """sketching.py:46-54 -- SeedSequence([seed, *idx]).generate_state(1, u64)[0]."""
    ent = [int(seed) & _M64] + [int(i) & _M64 for i in idx]
    return int(np.random.SeedSequence(entropy=ent).generate_state(1, np.uint64)[0])


def generator(seed: int) -> np.random.Generator:
    """sketching.py:57-58 -- default_rng(SeedSequence([seed & 2^64-1])) (PCG64)."""
    return np.random.default_rng(np.random.SeedSequence(entropy=[int(seed) & _M64]))


def pcg64_state(seed: int) -> tuple[int, int]:
    """128-bit (state, inc) of ``generator(seed)`` before its first draw."""
    st = generator(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


# --------------------------------------------------------------------------
# CountSketch draw (sketching.py:114-124, :141-150)
# --------------------------------------------------------------------------

def countsketch_numpy(seed: int, n: int, r: int, s: int):
    """sketching.py:141-150 via numpy itself: returns (cols int64 (n,s), signs f64 (n,s))."""
    rng = generator(seed)
    if s == 1:
        cols = rng.integers(0, r, size=(n, 1))
    else:
        keys = rng.random((n, r))
        cols = np.argpartition(keys, s - 1, axis=1)[:, :s]
    signs = rng.integers(0, 2, size=(n, s)).astype(np.float64) * 2.0 - 1.0
    return cols, signs


_CLIB = None


def _clib():
    """Build (if needed) and load oracle/countsketch.c -> oracle/build/libskp_oracle.so."""
    global _CLIB
    if _CLIB is not None:
        return _CLIB
    out_dir = os.path.join(_HERE, "build")
    so = os.path.join(out_dir, "libskp_oracle.so")
    src = os.path.join(_HERE, "countsketch.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        os.makedirs(out_dir, exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", so, src])
    lib = ctypes.CDLL(so)
    u64, i64 = ctypes.c_uint64, ctypes.c_int64
    lib.skpo_countsketch.argtypes = [u64, u64, u64, u64, i64, i64, ctypes.c_int32,
                                     ctypes.c_void_p, ctypes.c_void_p]
    lib.skpo_countsketch.restype = ctypes.c_int
    lib.skpo_pcg64_raw.argtypes = [u64, u64, u64, u64, i64, ctypes.c_void_p]
    lib.skpo_pcg64_advance.argtypes = [u64, u64, u64, u64, u64,
                                       ctypes.POINTER(u64), ctypes.POINTER(u64)]
    _CLIB = lib
    return lib


def _split(x: int):
    return (x >> 64) & _M64, x & _M64


def countsketch_c(seed: int, n: int, r: int, s: int):
    """Same draw as :func:`countsketch_numpy` through the plain-C restatement."""
    st, inc = pcg64_state(seed)
    cols = np.empty((n, s), dtype=np.int64)
    signs = np.empty((n, s), dtype=np.int8)
    rc = _clib().skpo_countsketch(*_split(st), *_split(inc), n, r, s,
                                  cols.ctypes.data, signs.ctypes.data)
    if rc != 0:
        raise ValueError("countsketch oracle: bad arguments")
    return cols, signs.astype(np.float64)


def pcg64_raw_c(st: int, inc: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    _clib().skpo_pcg64_raw(*_split(st), *_split(inc), count, out.ctypes.data)
    return out


def pcg64_advance_c(st: int, inc: int, delta: int) -> int:
    hi, lo = ctypes.c_uint64(), ctypes.c_uint64()
    _clib().skpo_pcg64_advance(*_split(st), *_split(inc), delta, ctypes.byref(hi), ctypes.byref(lo))
    return (hi.value << 64) | lo.value


class CountSketch:
    """The countsketch / identity branches of SketchOperator (sketching.py:93-213)."""

    def __init__(self, kind: str, n: int, r: int, seed: int, s: int | None = None):
        self.kind, self.n, self.r, self.seed = kind, int(n), int(r), int(seed) & _M64
        if kind == "countsketch":
            self.s = 1 if s is None else int(s)
            self.cols, self.signs = countsketch_numpy(self.seed, n, r, self.s)
            # CSR with data = signs/sqrt(s), indptr = arange(0, n*s+1, s)  (sketching.py:121-124)
            self.csr = sp.csr_array(((self.signs / math.sqrt(self.s)).ravel(), self.cols.ravel(),
                                     np.arange(0, n * self.s + 1, self.s)), shape=(n, r))
        elif kind == "identity":
            if r != n:
                raise ValueError("identity sketch needs r == n")
            self.s = None
        elif kind == "srht":              # sketching.py:125-130
            rng = generator(self.seed)
            self.n_pad = 1 << (int(n) - 1).bit_length()
            self.srht_signs = rng.integers(0, 2, size=self.n_pad).astype(np.float64) * 2.0 - 1.0
            self.subset = np.sort(rng.choice(self.n_pad, size=r, replace=False))
            self.s = None
        elif kind in ("gaussian", "sign"):  # sketching.py:131-136
            rng = generator(self.seed)
            if kind == "gaussian":
                self.dense = rng.standard_normal((n, r)) / math.sqrt(r)
            else:
                self.dense = (rng.integers(0, 2, size=(n, r)).astype(np.float64) * 2.0 - 1.0)
                self.dense /= math.sqrt(r)
            self.s = None
        else:
            raise ValueError(f"oracle covers countsketch/identity/srht/gaussian/sign, not {kind!r}")

    @staticmethod
    def fwht(a, axis: int = 0):
        """sketching.py:65-90: unnormalised Sylvester-ordered Walsh-Hadamard."""
        a = np.asarray(a, dtype=np.float64)
        if axis == 1:
            return CountSketch.fwht(a.T, 0).T
        n = a.shape[0]
        out = a.copy().reshape(n, -1)
        cols = out.shape[1]
        h = 1
        while h < n:
            out = out.reshape(n // (2 * h), 2, h, cols)
            out = np.stack((out[:, 0] + out[:, 1], out[:, 0] - out[:, 1]), axis=1).reshape(n, cols)
            h *= 2
        return out.reshape(a.shape)

    def apply_right(self, a):            # sketching.py:158-174
        a = as_matrix(a)
        if self.kind == "countsketch":
            return np.asarray(a @ self.csr)
        if self.kind == "srht":
            padded = np.zeros((a.shape[0], self.n_pad))
            padded[:, : self.n] = a
            return self.fwht(padded * self.srht_signs, 1)[:, self.subset] / math.sqrt(self.r)
        if self.kind in ("gaussian", "sign"):
            return a @ self.dense
        return a.copy()

    def apply_left_transpose(self, a):   # sketching.py:176-192
        a = as_matrix(a)
        if self.kind == "countsketch":
            return np.asarray(self.csr.T @ a)
        if self.kind == "srht":
            padded = np.zeros((self.n_pad, a.shape[1]))
            padded[: self.n, :] = a
            return self.fwht(padded * self.srht_signs[:, None], 0)[self.subset, :] / math.sqrt(self.r)
        if self.kind in ("gaussian", "sign"):
            return self.dense.T @ a
        return a.copy()

    def densify(self):                   # sketching.py:194-213
        if self.kind == "identity":
            return np.eye(self.n)
        if self.kind in ("gaussian", "sign"):
            return self.dense.copy()
        if self.kind == "srht":
            return self.apply_right(np.eye(self.n))
        out = np.zeros((self.n, self.r))
        out[np.repeat(np.arange(self.n), self.s), self.cols.ravel()] = self.signs.ravel() / math.sqrt(self.s)
        return out


def draw_omega(r1: int, r2: int, seed: int, kind: str = "gaussian") -> np.ndarray:
    """power.py:137-138: make_sketch(kind, r1, r2, seed).densify(); the
    Gaussian default is sketching.py:132-133, standard_normal((r1, r2)) / sqrt(r2)."""
    if kind == "gaussian":
        return generator(seed).standard_normal((r1, r2)) / math.sqrt(r2)
    return CountSketch(kind, r1, r2, seed).densify()


# --------------------------------------------------------------------------
# dense linalg (linalg.py:30-106)
# --------------------------------------------------------------------------

def as_matrix(a) -> np.ndarray:
    """linalg.py:30-39 (float64 cast, 2-D, non-empty, finite)."""
    out = np.asarray(a, dtype=np.float64)
    if out.ndim != 2 or out.size == 0 or not np.all(np.isfinite(out)):
        raise ValueError("matrix must be 2-D, non-empty and finite")
    return out


def orthonormalize(y, tol=None) -> np.ndarray:
    """linalg.py:57-81: pivoted economy QR, keep |R_ii| >= max(m,c)*eps*max|R_ii|."""
    y = as_matrix(y)
    tol = max(y.shape) * np.finfo(np.float64).eps if tol is None else tol
    q, r, _ = sla.qr(y, mode="economic", pivoting=True)
    d = np.abs(np.diag(r))
    if d.max() == 0.0:
        raise ValueError("cannot orthonormalize an all-zero matrix")
    return np.ascontiguousarray(q[:, : int(np.count_nonzero(d >= tol * d.max()))])


def thin_svd(a):
    """linalg.py:84-88 (LAPACK gesdd): (U, sigma, V)."""
    u, s, vh = sla.svd(as_matrix(a), full_matrices=False)
    return u, s, vh.T.copy()


def pinv(m, rel_tol=None):
    """linalg.py:91-106."""
    m = as_matrix(m)
    rel_tol = max(m.shape) * np.finfo(np.float64).eps if rel_tol is None else rel_tol
    u, s, v = thin_svd(m)
    if s[0] == 0.0:
        return np.zeros((m.shape[1], m.shape[0]))
    inv = np.where(s > rel_tol * s[0], 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return (v * inv) @ u.T


# --------------------------------------------------------------------------
# power methods (power.py:49-298)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Spec:
    """The fields of RangeFinderSpec (power.py:49-77) the hot path reads."""
    k: int
    l: int
    r1: int
    r2: int
    q: int
    eps: float = 0.5
    sketch_kind: str = "countsketch"
    seed: int = 0
    stabilized: bool = True
    s: int = 1
    omega_kind: str = "gaussian"
    s2_kind: str | None = None
    s2_r: int | None = None


def power_iterate(atil, omega, q: int, stabilized: bool = True):
    """power.py:113-134."""
    atil, omega = as_matrix(atil), as_matrix(omega)
    y = atil @ omega
    for _ in range(q):
        if stabilized:
            y = orthonormalize(y)
        y = atil @ (atil.T @ y)
    return y


def range_finder_sketched(a, spec: Spec, timings: dict | None = None):
    """power.py:141-154 (Alg. 1), with optional per-phase wall times."""
    import time
    t = [time.perf_counter()]
    a = as_matrix(a)
    t.append(time.perf_counter())
    m, n = a.shape
    sk = CountSketch(spec.sketch_kind, n, spec.r1, substream(spec.seed, 0), s=spec.s)
    t.append(time.perf_counter())
    omega = draw_omega(spec.r1, spec.r2, substream(spec.seed, 1), spec.omega_kind)
    t.append(time.perf_counter())
    atil = sk.apply_right(a)
    t.append(time.perf_counter())
    y = power_iterate(atil, omega, spec.q, stabilized=spec.stabilized)
    t.append(time.perf_counter())
    qb = orthonormalize(y)
    t.append(time.perf_counter())
    if timings is not None:
        for name, i in (("cast", 1), ("make_sketch", 2), ("omega", 3), ("apply_right", 4),
                        ("power", 5), ("orth", 6)):
            timings[name] = timings.get(name, 0.0) + t[i] - t[i - 1]
    return qb


def randsvd(a, qb):
    """power.py:181-199 (orthonormality check 1e-6, B = Q^T a, gesdd)."""
    a, qb = as_matrix(a), as_matrix(qb)
    if np.abs(qb.T @ qb - np.eye(qb.shape[1])).max() > 1e-6:
        raise ValueError("Q is not orthonormal")
    u, s, v = thin_svd(qb.T @ a)
    return qb @ u, s, v


def lowrank_factorize(a, spec: Spec):
    """power.py:202-239: Y = powered block, X = pinv(S2^T Y) (S2^T a), S2 ~ substream(seed, 2)."""
    a = as_matrix(a)
    m, n = a.shape
    s1 = CountSketch(spec.sketch_kind, n, spec.r1, substream(spec.seed, 0), s=spec.s)
    atil = s1.apply_right(a)
    omega = draw_omega(spec.r1, spec.r2, substream(spec.seed, 1), spec.omega_kind)
    y = power_iterate(atil, omega, spec.q, stabilized=spec.stabilized)
    s2 = CountSketch(spec.s2_kind or spec.sketch_kind, m, spec.s2_r or spec.r1,
                     substream(spec.seed, 2), s=spec.s)
    return y, pinv(s2.apply_left_transpose(y)) @ s2.apply_left_transpose(a)


def nystrom_core(a, spec: Spec, stabilized: bool = False, timings: dict | None = None):
    """power.py:272-287 without _check_psd (O(n^3), infeasible at C4).

    ``stabilized=False`` is the literal reference (Y = W~^q Omega).
    ``stabilized=True`` orthonormalises between W~ products -- same span in
    exact arithmetic; the parity reference for FP32.
    ``timings`` (optional): seconds per phase (apply_right = K S, left_t =
    S^T C~, core = the l-dimensional power + W, contract = C~ Y).
    Returns (C, W).
    """
    import time
    t = {} if timings is None else timings
    t0 = time.perf_counter()
    a = as_matrix(a)
    n = a.shape[0]
    sk = CountSketch(spec.sketch_kind, n, spec.r1, substream(spec.seed, 0), s=spec.s)
    ctil = sk.apply_right(a)
    t1 = time.perf_counter()
    wtil = sk.apply_left_transpose(ctil)
    wtil = (wtil + wtil.T) / 2.0
    t2 = time.perf_counter()
    y = draw_omega(spec.r1, spec.r2, substream(spec.seed, 1), spec.omega_kind)
    for _ in range(spec.q):
        if stabilized:
            y = orthonormalize(y)
        y = wtil @ y
    w = y.T @ (wtil @ y)
    t3 = time.perf_counter()
    c = ctil @ y
    t4 = time.perf_counter()
    t.update(apply_right=t1 - t0, left_t=t2 - t1, core=t3 - t2, contract=t4 - t3)
    return c, (w + w.T) / 2.0


def proj_rel_error(a, qb) -> float:
    """||A - QQ^T A||_F / ||A||_F (diagnostics.py:159-166, Frobenius part), exact."""
    a = as_matrix(a)
    r = a - qb @ (qb.T @ a)
    return float(np.linalg.norm(r) / np.linalg.norm(a))


def nystrom_rel_error(a, c, w) -> float:
    """||A - C W^+ C^T||_F / ||A||_F."""
    a = as_matrix(a)
    return float(np.linalg.norm(a - c @ pinv(w) @ c.T) / np.linalg.norm(a))
