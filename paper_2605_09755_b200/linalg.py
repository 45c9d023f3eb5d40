"""Dense linalg on the B200 (drop-in for skpower.linalg, reference linalg.py).

``orthonormalize`` is CholeskyQR2 with a rank-revealing eigen pass
(replaces the pivoted QR of linalg.py:57-81); ``thin_svd`` / ``pinv`` run
the one-sided Jacobi SVD in fp64 on the matrix itself (replace LAPACK
gesdd, linalg.py:84-106): no Gram matrix, so cond 1e12 inputs keep their
small singular values.  (randsvd's r2 x n core keeps the Gram route, whose
eigen-decomposition of B B^T resolves sigma_i >~ 1e-8 sigma_1 -- DESIGN.md.)
Results follow the operand kind (numpy in -> numpy out, CUDA tensor in ->
CUDA tensor out).
"""
from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _convert, _engine, _ops
from ._ops import F32, F64


class SvdResult(NamedTuple):
    """Thin SVD A = U diag(sigma) V^T (linalg.py:18-27)."""
    U: object
    sigma: object
    V: object


def _backend(dtype, device):
    return _ops.CudaBackend(device, dtype)


def as_matrix(a, name: str = "matrix"):
    """Validate a 2-D, non-empty, finite operand (linalg.py:30-39).

    numpy input returns a float64 numpy array like the reference; tensors are
    validated on their device and returned as float32/float64 tensors."""
    if isinstance(a, torch.Tensor):
        return _convert.upload(a, name, a.device if a.is_cuda else None).t
    out = np.asarray(a, dtype=np.float64)
    if out.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={out.ndim}")
    if out.size == 0:
        raise ValueError(f"{name} must be non-empty")
    op = _convert.upload(out, name)
    del op
    return out


def matmul(a, b):
    """a @ b with a dimension check (linalg.py:42-48)."""
    oa, ob = _convert.upload(a, "a"), _convert.upload(b, "b", _ops.require_cuda())
    if oa.t.shape[1] != ob.t.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(oa.t.shape)} @ {tuple(ob.t.shape)}")
    dt = _convert.common_dtype(oa, ob)
    out = _ops.gemm(_convert.as_dtype(oa, dt), _convert.as_dtype(ob, dt))
    return _convert.download(out, oa.kind)


def orthonormalize(y, tol: float | None = None):
    """Orthonormal basis for range(y), numerically rank-truncated (linalg.py:57-81).

    The reference's pivoted QR runs in fp64 for every input: an fp32 y whose
    rank decision the fp32 CholeskyQR cuts short (it resolves ~2.8e-6 of
    sigma_1, fp32 rounding noise included) is redone in fp64, so the column
    count follows the reference (power._promote_range_finder's rule)."""
    op = _convert.upload(y, "y")
    be = _backend(op.t.dtype, op.t.device)
    q = _engine.orthonormalize(be, _engine.LOCAL, op.t, tol=tol)
    if op.t.dtype == _ops.F32 and q.shape[1] < min(op.t.shape):
        t64 = _ops.cast(op.t, _ops.F64)
        q = _engine.orthonormalize(_backend(_ops.F64, op.t.device), _engine.LOCAL, t64, tol=tol)
    return _convert.download(q, op.kind)


def _thin_svd_dev(be, a: torch.Tensor):
    """(U, sigma, V) of a (p x q) by one-sided Jacobi on a (p >= q) or a^T;
    fp64 results, cast to the compute dtype for U and V."""
    p, q = a.shape
    if p >= q:
        u, s, v = _ops.gesvj(a)
    else:
        v, s, u = _ops.gesvj(a.T.contiguous())
    return be.to_compute(u), s, be.to_compute(v)


def thin_svd(a) -> SvdResult:
    """Economy SVD with descending singular values (linalg.py:84-88)."""
    op = _convert.upload(a, "a")
    be = _backend(op.t.dtype, op.t.device)
    u, s, v = _thin_svd_dev(be, op.t)
    return SvdResult(_convert.download(u, op.kind), _convert.download(s, op.kind),
                     _convert.download(v, op.kind))


def _pinv_dev(be, m: torch.Tensor, rel_tol=None):
    if rel_tol is None:
        rel_tol = max(m.shape) * np.finfo(np.float64).eps
    u, s, v = _thin_svd_dev(be, m)
    s0 = float(s[0].item())
    if s0 == 0.0:
        return torch.zeros((m.shape[1], m.shape[0]), dtype=m.dtype, device=m.device)
    inv = torch.where(s > rel_tol * s0, 1.0 / torch.where(s > 0, s, torch.ones_like(s)),
                      torch.zeros_like(s))
    vs = v.clone()
    be.scale_cols_(vs, inv)
    return be.mm(vs, u, tb=True)


def pinv(m, rel_tol: float | None = None):
    """Moore-Penrose pseudoinverse via the thin SVD (linalg.py:91-106)."""
    op = _convert.upload(m, "m")
    be = _backend(op.t.dtype, op.t.device)
    return _convert.download(_pinv_dev(be, op.t, rel_tol), op.kind)


def frobenius_norm(a) -> float:
    op = _convert.upload(a, "a")
    return float(np.sqrt(_ops.sumsq(op.t).item()))


def spectral_norm(a) -> float:
    op = _convert.upload(a, "a")
    be = _backend(op.t.dtype, op.t.device)
    t = op.t if op.t.shape[0] <= op.t.shape[1] else op.t.T.contiguous()
    w, _ = be.eig_desc64(be.gram64_rows(t))
    return float(np.sqrt(max(float(w[0].item()), 0.0)))


def norms(a) -> tuple[float, float]:
    return spectral_norm(a), frobenius_norm(a)
