"""Backend-agnostic orchestration of the sketched power method.

The algorithm (reference power.py:113-154, :181-199, :258-298 and
linalg.py:57-88) written once against two small interfaces:

* a compute backend ``be`` (``_ops.CudaBackend`` in the product: every call is
  a libskp kernel) providing mm / gram64 / chol_inv64 / eig_desc64 / ...;
* a communicator ``comm`` with ``allreduce_(t)`` (in-place sum over ranks)
  for row-sharded runs: A, A.S and Y live as row slabs, and only the l x r2
  product A~^T Y, the r2 x r2 Gram matrices and the r2 x n matrix Q^T A are
  summed.

Orthonormalisation is CholeskyQR2 (two passes of Gram -> Cholesky -> L^{-1}
-> Y L^{-T}).  Where the reference's pivoted QR would drop columns
(linalg.py:75-81) the Cholesky pivot check fails and an eigen-based
truncating pass (Y V_k Lambda_k^{-1/2}) runs first.
"""
from __future__ import annotations

import numpy as np


class LocalComm:
    rank = 0
    world = 1

    def allreduce_(self, t):
        return t


LOCAL = LocalComm()

# Relative pivot floor for the Gram-based rank test: CholeskyQR resolves
# sigma_i / sigma_1 down to ~sqrt(eps) of the Gram's precision, so the
# reference tolerance max(m, c) * eps (linalg.py:51-54) is raised to these
# floors (documented deviation).
PIVOT_FLOOR = {"float64": 1e-6, "float32": 5e-4}
ORTHO_TOL = {"float64": 1e-6, "float32": 1e-4}


def _dtype_key(be) -> str:
    return "float32" if "32" in str(be.dtype) else "float64"


def pivot_tol(be, rows: int, cols: int, tol=None) -> float:
    ref = (max(rows, cols) * np.finfo(np.float64).eps) if tol is None else float(tol)
    return max(ref, PIVOT_FLOOR[_dtype_key(be)])


def orthonormalize(be, comm, y, tol=None, rows_total: int | None = None, lazy: bool = False,
                   passes: int = 2, planes_out: bool = False):
    """Orthonormal basis of range(y) (linalg.py:57-81) by CholeskyQR2.

    ``lazy``: no host synchronisation; a Cholesky failure (rank deficiency)
    is only flagged on the device (``be.lazy_failed()``) and the caller must
    redo the computation eagerly, where the truncating eigen path runs.
    ``passes=1`` (lazy only): one CholeskyQR pass -- same span, orthogonality
    ~eps * cond(Y)^2; used for the stabilisations inside the power iteration,
    whose only job is to keep the block well conditioned (the final Q always
    gets two passes)."""
    if hasattr(be, "orth_planes") and not isinstance(y, np.ndarray) and hasattr(y, "hi"):
        # y given as the fp16 planes of its transpose (the lazy planes path)
        rows_total = y.cols if rows_total is None else rows_total
        rel = pivot_tol(be, rows_total, y.rows, tol)
        if lazy and passes == 2:
            return be.orth_planes(comm, y, rel, planes_out)
        y = be.planes_to_compute(y)
    c = y.shape[1]
    rows_total = y.shape[0] if rows_total is None else rows_total
    rel = pivot_tol(be, rows_total, c, tol)
    g = comm.allreduce_(be.gram64(y))
    if lazy:
        x = be.chol_inv64(g, rel, lazy=True)
        q = be.mm(y, be.to_compute(x), tb=True)
        if passes == 1:
            return q
        g2 = comm.allreduce_(be.gram64(q, accurate=True))
        x2 = be.chol_inv64(g2, 0.0, lazy=True)
        return be.mm(q, be.to_compute(x2), tb=True)
    x = be.chol_inv64(g, rel)
    if x is None:
        w, v = be.eig_desc64(g)
        t, k = be.eig_orth64(w, v, rel * rel)
        if k == 0:
            raise ValueError("cannot orthonormalize an all-zero matrix")
        y = be.mm(y, be.to_compute(be.cols(t, k)))
        g = comm.allreduce_(be.gram64(y))
        x = be.chol_inv64(g, 0.0)
        if x is None:
            raise RuntimeError("orthonormalize: Cholesky failed after rank truncation")
    q = be.mm(y, be.to_compute(x), tb=True)
    g2 = comm.allreduce_(be.gram64(q, accurate=True))
    x2 = be.chol_inv64(g2, 0.0)
    if x2 is None:
        raise RuntimeError("orthonormalize: second CholeskyQR pass failed")
    return be.mm(q, be.to_compute(x2), tb=True)


def power_iterate(be, comm, atil, omega, q: int, stabilized: bool = True, rows_total=None,
                  lazy: bool = False):
    """power.py:113-134 on a row slab of A~: Y = A~ Omega, then q x
    {orth(Y) if stabilized; Z = sum_p A~_p^T Y_p; Y = A~ Z}.  A~ feeds all
    1 + 2q products, so it is prepared once (be.prepare: the fp16 split of
    the 3xFP16 GEMM on the CUDA backend)."""
    atil = be.prepare(atil)
    if lazy and stabilized and q > 0 and hasattr(be, "planes_ok") and be.planes_ok(atil, omega):
        def rel_of(yt):
            return pivot_tol(be, yt.cols if rows_total is None else rows_total, yt.rows)
        return be.power_lazy_planes(comm, atil, omega, q, rel_of)
    y = be.mm(atil, omega)
    for _ in range(q):
        if stabilized:
            y = orthonormalize(be, comm, y, rows_total=rows_total, lazy=lazy,
                               passes=1 if lazy else 2)
        z = comm.allreduce_(be.mm(atil, y, ta=True))
        y = be.mm(atil, z)
    return y


def randsvd(be, comm, a, qb, check: bool = True, amax_hint=None):
    """power.py:181-199: B = Q^T A (summed over row slabs), thin SVD of B via
    the fp64 Gram B B^T and the eigensolver; U = Q U~, V = B^T U~ / sigma.

    B is formed transposed, B^T = A^T Q (n x c): the long dimension n then
    sits on the GEMM's M side (full 256-row CTA-pair tiles) instead of the
    short c, and B B^T = (B^T)^T B^T, V = B^T U~ read it directly."""
    if check:
        g = comm.allreduce_(be.gram64(be.dense(qb) if hasattr(be, "dense") else qb))
        dev = be.orth_dev(g)
        if not dev <= ORTHO_TOL[_dtype_key(be)]:
            raise ValueError(f"Q is not orthonormal (deviation {dev:.3e})")
    out = _randsvd_core(be, comm, be.mm_at_big(a, qb, amax_hint), qb)   # B^T: this rank's part
    if be.overflowed(comm):
        # the in-kernel fp16 split met an entry beyond its exponent bound (a
        # hint that did not hold): recompute with 3xTF32 on every rank.  The
        # flag is read once, after everything is queued (no mid-call sync).
        out = _randsvd_core(be, comm, be.mm(a, be.dense(qb), ta=True), qb)
    return out


def _randsvd_core(be, comm, bt, qb):
    bt = comm.allreduce_(bt)
    n, c = bt.shape
    gb = be.gram64_rows_t(bt)                               # c x c, fp64
    w, v = be.eig_desc64(gb)
    p = min(c, n)
    sig, inv = be.sqrt_eigs(w)
    vc = be.to_compute(be.cols(v, p))
    planes = hasattr(qb, "hi")          # Q given as the fp16 planes of Q^T
    u = be.mm(qb, vc, ta=planes)
    vv = be.mm(bt, vc)
    be.scale_cols_(vv, inv[:p])
    return u, sig[:p], vv


def nystrom(be, comm, ctil, wtil, omega, q: int, stabilized: bool):
    """power.py:276-287 given C~ (row slab) and the summed, symmetrised W~."""
    y = omega
    for _ in range(q):
        if stabilized:
            y = orthonormalize(be, LOCAL, y)
        y = be.mm(wtil, y)
    cmat = be.mm(ctil, y)
    w = be.mm(y, be.mm(wtil, y), ta=True)
    be.symmetrize_(w)
    return cmat, w
