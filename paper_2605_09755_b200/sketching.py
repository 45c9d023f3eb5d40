"""Seeded sketch operators on the B200 (drop-in for skpower.sketching).

Mirrors /root/reference/pkg/src/skpower/sketching.py: ``SketchOperator``
(:93), ``make_sketch`` (:216), ``substream`` (:46), the functional forms
(:225-237) and ``SKETCH_KINDS`` (:39).

* ``countsketch`` -- S is regenerated ON THE DEVICE from the seed by the K1
  kernel, bit-exact with the reference's numpy draw (sketching.py:141-150);
  apply_right / apply_left_transpose are the K2 / K3 gather kernels.
* ``identity``    -- the classical (unsketched) hook (sketching.py:137-139).
* ``gaussian`` / ``sign`` -- dense S drawn on the host with the reference's
  numpy stream (bit-identical), applied with the device GEMM.
* ``srht``        -- the signs and the sorted coordinate subset are numpy's
  draw (bit-identical, sketching.py:125-130); apply_right /
  apply_left_transpose are the K7 kernel (sign, zero-pad, fast
  Walsh-Hadamard transform in shared memory, subset gather), densify is K7
  applied to the identity.  No CPU fallback exists.
"""
from __future__ import annotations

import math
import threading

import numpy as np
import torch

from . import _convert, _ops
from ._ops import F32, F64

SKETCH_KINDS = ("gaussian", "sign", "countsketch", "srht", "identity")
DEVICE_KINDS = ("gaussian", "sign", "countsketch", "srht", "identity")

_DENSIFY_CAP = 10**7
_MASK64 = (1 << 64) - 1


def substream(seed: int, *indices: int) -> int:
    """Independent 64-bit seed from (seed, *indices) -- sketching.py:46-54.
    Host-side seed expansion (numpy SeedSequence), as in the reference."""
    entropy = [int(seed) & _MASK64] + [int(i) & _MASK64 for i in indices]
    return int(np.random.SeedSequence(entropy=entropy).generate_state(1, np.uint64)[0])


def _host_rng(seed: int) -> np.random.Generator:
    # sketching.py:57-58
    return np.random.default_rng(np.random.SeedSequence(entropy=[int(seed) & _MASK64]))


def pcg64_state(seed: int) -> tuple[int, int]:
    """128-bit PCG64 (state, inc) that _rng(seed) starts from (passed to K1)."""
    st = _host_rng(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


class SketchOperator:
    """Immutable seeded linear map from n to r coordinates (device resident).

    Same constructor, attributes (kind, n, r, seed, s) and methods as the
    reference; ``_cols`` / ``_signs`` are host copies of the device arrays
    (int64 / float64 +-1, as the reference stores them).
    """

    def __init__(self, kind: str, n: int, r: int, seed: int, s: int | None = None, device=None):
        if kind not in SKETCH_KINDS:
            raise ValueError(f"unknown sketch kind {kind!r}, expected one of {SKETCH_KINDS}")
        if r < 1:
            raise ValueError(f"sketch dimension r must be >= 1, got {r}")
        if n < 1:
            raise ValueError(f"input dimension n must be >= 1, got {n}")
        self.kind = kind
        self.n = int(n)
        self.r = int(r)
        self.seed = int(seed) & _MASK64
        self.s = None
        self._dense_host = None
        self._dense_dev = {}
        self.device = _ops.require_cuda(device)
        if kind == "srht":  # (handled first; the chain below covers the other kinds)
            n_pad = 1 << (int(n) - 1).bit_length()
            if r > n_pad:
                raise ValueError(f"srht needs r <= padded dimension {n_pad}, got r={r}")
            rng = _host_rng(self.seed)
            self._n_pad = n_pad
            self._srht_signs = rng.integers(0, 2, size=n_pad).astype(np.float64) * 2.0 - 1.0
            self._subset = np.sort(rng.choice(n_pad, size=r, replace=False))
            self.d_srht_signs = torch.from_numpy(self._srht_signs.astype(np.int8)).to(self.device)
            self.d_subset = torch.from_numpy(self._subset.astype(np.int32)).to(self.device)
        if kind == "countsketch":
            s = 1 if s is None else int(s)
            if not 1 <= s <= r:
                raise ValueError(f"countsketch needs 1 <= s <= r, got s={s}, r={r}")
            self.s = s
            st, inc = pcg64_state(self.seed)
            self.d_cols, self.d_signs = _ops.countsketch(st, inc, self.n, self.r, s, self.device)
            self.colptr, self.entries = _ops.csc(self.d_cols, self.d_signs, self.n, s, self.r)
        elif kind == "gaussian":
            self._dense_host = _host_rng(self.seed).standard_normal((n, r)) / math.sqrt(r)
        elif kind == "sign":
            d = _host_rng(self.seed).integers(0, 2, size=(n, r)).astype(np.float64) * 2.0 - 1.0
            self._dense_host = d / math.sqrt(r)
        elif kind == "identity":
            if r != n:
                raise ValueError(f"identity sketch needs r == n, got n={n}, r={r}")

    def __repr__(self):
        extra = f", s={self.s}" if self.kind == "countsketch" else ""
        return f"SketchOperator({self.kind}, n={self.n}, r={self.r}, seed={self.seed}{extra})"

    # reference-compatible host views of the draw
    @property
    def _cols(self) -> np.ndarray:
        return self.d_cols.cpu().numpy().astype(np.int64)

    @property
    def _signs(self) -> np.ndarray:
        if self.kind == "srht":
            return self._srht_signs
        return self.d_signs.cpu().numpy().astype(np.float64)

    def _dense(self, dtype) -> torch.Tensor:
        t = self._dense_dev.get(dtype)
        if t is None:
            t = torch.from_numpy(self._dense_host).to(self.device, dtype=dtype)
            self._dense_dev[dtype] = t
        return t

    # -- device-level application (tensors in, tensors out) -----------------
    def right(self, a: torch.Tensor, out=None, fro2=None, nonfinite=None) -> torch.Tensor:
        if self.kind == "countsketch":
            # fp32: the row gather (K2 v2) and an in-place column un-permutation
            # (C5's shape: 171 + 11 ms against 623 ms for K2 v1); K2 v1 when the
            # gather's plan or shape does not apply
            if (a.dtype == torch.float32 and self.r <= _ops.UNPERMUTE_MAX_COLS
                    and (out is None or (out.stride(1) == 1 and out.dtype == a.dtype))):
                got = self.right_permuted(a, out=out, fro2=fro2, nonfinite=nonfinite)
                if got is not None:
                    return _ops.unpermute_cols(got[0], got[1])
            return _ops.sketch_right(a, self.colptr, self.entries, self.s, self.r, out, fro2,
                                     nonfinite)
        if fro2 is not None or nonfinite is not None:
            _ops.sumsq(a, fro2, nonfinite)
        if self.kind == "identity":
            return a.clone() if out is None else out.copy_(a)
        if self.kind == "srht":
            return _ops.srht(a, self.d_srht_signs, self._n_pad, self.d_subset, self.r, False, out)
        return _ops.gemm(a, self._dense(a.dtype), out=out)

    def gather_plan(self, check: bool = True):
        """Cached K2 v2 plan: (plan, perm) -- perm (numpy) only after the host
        check -- or None when the kernel does not apply (check=True also
        returns None for a schedule that overflowed)."""
        if self.kind != "countsketch":
            return None
        if not hasattr(self, "_gather"):
            self._gather = _ops.gather_plan(self.colptr, self.entries, self.n, self.r,
                                            self.device, check=check)
        if check and self._gather is not None and self._gather[1] is None:
            self._gather = _ops.gather_plan_checked(self._gather[0], self.r)
        return self._gather

    def right_permuted(self, a: torch.Tensor, out=None, fro2=None, nonfinite=None,
                       deferred: bool = False, amax=None, out_dtype=None):
        """(a @ S P, perm) with perm[v] (int32, on the device) = the column of
        a @ S at position v, via the row-gather kernel (fp32, n <= 98304); None
        when it does not apply.  deferred=True skips the plan's host check: a
        failed schedule then adds _ops.GATHER_PLAN_FAIL_MARK to *nonfinite
        (required) and writes nothing -- the caller falls back to right().
        Range-finder use: (a S P)(P^T Omega) == (a S) Omega.  amax: see
        _ops.sketch_gather."""
        if a.dtype != torch.float32 or (a.stride(0) * 4) % 16 or a.data_ptr() % 16:
            return None
        if deferred and nonfinite is None:
            raise ValueError("right_permuted(deferred=True) needs the nonfinite counter")
        plan = self.gather_plan(check=not deferred)
        if plan is None:
            return None
        g = plan[0]
        perm_dev = g[:4 * self.r].view(torch.int32)   # the first r entries are the valid ones
        return (_ops.sketch_gather(a, g, self.r, self.s, out, fro2, nonfinite, amax, out_dtype),
                perm_dev)

    def left_t(self, x: torch.Tensor, out=None) -> torch.Tensor:
        if self.kind == "countsketch":
            return _ops.sketch_left_t(x, self.colptr, self.entries, self.s, self.r, out)
        if self.kind == "identity":
            return x.clone() if out is None else out.copy_(x)
        if self.kind == "srht":
            return _ops.srht(x, self.d_srht_signs, self._n_pad, self.d_subset, self.r, True, out)
        return _ops.gemm(self._dense(x.dtype), x, ta=True, out=out)

    # -- reference API --------------------------------------------------------
    def apply_right(self, a):
        """a @ S for a with n columns (sketching.py:158-174)."""
        op = _convert.upload(a, "a", self.device)
        if op.t.shape[1] != self.n:
            raise ValueError(f"dimension mismatch: a has {op.t.shape[1]} cols, sketch n={self.n}")
        return _convert.download(self.right(op.t), op.kind)

    def apply_left_transpose(self, a):
        """S.T @ a for a with n rows (sketching.py:176-192)."""
        op = _convert.upload(a, "a", self.device)
        if op.t.shape[0] != self.n:
            raise ValueError(f"dimension mismatch: a has {op.t.shape[0]} rows, sketch n={self.n}")
        return _convert.download(self.left_t(op.t), op.kind)

    def densify(self) -> np.ndarray:
        """Explicit n x r matrix (host numpy, test oracle) -- sketching.py:194-213."""
        if self.n * self.r > _DENSIFY_CAP:
            raise ValueError(f"densify cap exceeded: {self.n} x {self.r} > {_DENSIFY_CAP} entries")
        if self.kind == "countsketch":
            out = np.zeros((self.n, self.r))
            rows = np.repeat(np.arange(self.n), self.s)
            out[rows, self._cols.ravel()] = self._signs.ravel() / math.sqrt(self.s)
            return out
        if self.kind == "identity":
            return np.eye(self.n)
        if self.kind == "srht":   # S = (S^T I)^T, K7 on the identity
            eye = torch.eye(self.n, dtype=F64, device=self.device)
            return self.left_t(_ops.aligned2d(eye)).T.cpu().numpy().copy()
        return self._dense_host.copy()


def make_sketch(kind: str, n: int, r: int, seed: int, s: int | None = None,
                device=None) -> SketchOperator:
    """Construct a sketch operator; deterministic in (kind, n, r, seed) -- sketching.py:216-222."""
    return SketchOperator(kind, n, r, seed, s=s, device=device)


def apply_right(a, sketch: SketchOperator):
    return sketch.apply_right(a)


def apply_left_transpose(sketch: SketchOperator, a):
    return sketch.apply_left_transpose(a)


def densify(sketch: SketchOperator) -> np.ndarray:
    return sketch.densify()


def draw_omega(kind: str, rows: int, cols: int, seed: int) -> np.ndarray:
    """The start block (power.py:137-138): host numpy draw, bit-identical to the
    reference (the ziggurat's data-dependent stream stays on the host)."""
    if kind == "gaussian":
        return _host_rng(seed).standard_normal((rows, cols)) / math.sqrt(cols)
    if kind == "sign":
        d = _host_rng(seed).integers(0, 2, size=(rows, cols)).astype(np.float64) * 2.0 - 1.0
        return d / math.sqrt(cols)
    if kind == "identity":
        if rows != cols:
            raise ValueError(f"identity sketch needs r == n, got n={rows}, r={cols}")
        return np.eye(rows)
    if kind in ("countsketch", "srht"):
        # (the reference's own route for every family: make_sketch(...).densify(),
        # with its densify cap)
        return make_sketch(kind, rows, cols, seed).densify()
    raise ValueError(f"unsupported omega kind {kind!r} on the B200 path")


def omega_device(kind: str, rows: int, cols: int, seed: int, dtype, device, perm_dev=None,
                 fail_counter=None):
    """The Gaussian start block drawn ON THE DEVICE (numpy's ziggurat
    reproduced draw for draw, omega.cu), with P^T applied when perm_dev is
    given; None for the other kinds (drawn on the host).  A generation that
    could not complete adds _ops.OMEGA_FAIL_MARK to fail_counter."""
    if kind != "gaussian":
        return None
    st, inc = pcg64_state(seed)
    om = _ops.gaussian(st, inc, rows, cols, math.sqrt(cols), dtype, device, fail_counter)
    return _ops.permute_rows(om, perm_dev) if perm_dev is not None else om


class OmegaDraw:
    """The host-side Omega draw (numpy, bit-identical to the reference) on a
    background thread -- numpy's generator fills release the GIL -- so it
    overlaps the device's sketch; to_device() joins, uploads (pinned,
    asynchronous) and optionally applies P^T on the device."""

    def __init__(self, kind: str, rows: int, cols: int, seed: int, dtype):
        self.rows, self.cols, self.dtype = rows, cols, dtype
        self._host = None
        self._err = None
        self._t = threading.Thread(target=self._run, args=(kind, seed), daemon=True)
        self._t.start()

    def _run(self, kind, seed):
        try:
            om = draw_omega(kind, self.rows, self.cols, seed)
            host = torch.from_numpy(om.astype(np.float32) if self.dtype == F32 else om)
            self._host = host.pin_memory() if self.rows * self.cols > 1 << 16 else host
        except BaseException as e:  # re-raised on the caller's thread
            self._err = e

    def to_device(self, device, perm_dev: torch.Tensor | None = None) -> torch.Tensor:
        self._t.join()
        if self._err is not None:
            raise self._err
        out = _ops.empty2d(self.rows, self.cols, self.dtype, device)
        out.copy_(self._host, non_blocking=True)
        if perm_dev is not None:
            out = _ops.permute_rows(out, perm_dev)
        return out


def omega_tensor(kind: str, rows: int, cols: int, seed: int, dtype, device,
                 row_perm: np.ndarray | None = None) -> torch.Tensor:
    """Omega on the device with 16-byte-aligned rows (TMA operand); with
    row_perm, P^T Omega (rows reordered on the host before the upload)."""
    om = draw_omega(kind, rows, cols, seed)
    if row_perm is not None:
        om = om[row_perm]
    out = _ops.empty2d(rows, cols, dtype, device)
    host = torch.from_numpy(om.astype(np.float32) if dtype == F32 else om)
    if rows * cols > 1 << 16:
        host = host.pin_memory()
    out.copy_(host, non_blocking=True)
    return out
