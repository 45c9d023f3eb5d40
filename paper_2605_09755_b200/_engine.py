"""Backend-agnostic orchestration of the sketched power method.

The algorithm (reference power.py:113-154, :181-199, :258-298 and
linalg.py:57-88) written once against two small interfaces:

* a compute backend ``be`` (``_ops.CudaBackend`` in the product: every call is
  a libskp kernel) providing mm / gram64 / chol_inv64 / eig_desc64 / ...;
* a communicator ``comm`` with ``allreduce_(t)`` (in-place sum over ranks)
  for row-sharded runs: A, A.S and Y live as row slabs, and only the l x r2
  product A~^T Y, the r2 x r2 Gram matrices and the r2 x n matrix Q^T A are
  summed.

Orthonormalisation is shifted CholeskyQR3 (three passes of Gram ->
Cholesky -> L^{-1} -> Y L^{-T}, the first on a shifted Gram).  Where the
reference's pivoted QR would drop columns (linalg.py:75-81) the second
pass's pivot check fails and an eigen-based truncating step
(Q V_k Lambda_k^{-1/2}) runs before the last pass.
"""
from __future__ import annotations

import numpy as np


class LocalComm:
    rank = 0
    world = 1

    def allreduce_(self, t):
        return t


LOCAL = LocalComm()

# Orthonormalisation is shifted CholeskyQR3 (Fukaya et al., SIAM J. Sci.
# Comput. 2020): pass 1 factors G + SHIFT_REL * max_i G_ii * I, which never
# fails on a numerically full-rank Y and leaves range(Y) intact (directions
# below the shift come out damped, not dropped); passes 2 and 3 are plain
# CholeskyQR on the now well-conditioned block.  The rank test (the
# reference's |R_ii| >= tol * max|R_ii|, linalg.py:75-81) runs on pass 2's
# Gram, where a direction with sigma_i(Y)/sigma_1(Y) = rho < sqrt(shift)
# has pivot rho / sqrt(shift): its smallest resolvable pivot ratio is
# RESOLVE (set by the Gram's own rounding), so the smallest resolvable rho
# is RESOLVE * sqrt(SHIFT_REL) -- 2.8e-6 in fp32 and 3.2e-13 in fp64, where
# the reference keeps max(m, c) * eps (5.8e-11 at C3).
SHIFT_REL = {"float64": 1e-13, "float32": 2.0 ** -17}
RESOLVE = {"float64": 1e-6, "float32": 1e-3}
ORTHO_TOL = {"float64": 1e-6, "float32": 1e-4}


def _dtype_key(be) -> str:
    return "float32" if "32" in str(be.dtype) else "float64"


def rank_floor(be, rows: int, cols: int, tol=None) -> float:
    """Smallest kept sigma_i(Y) / sigma_1(Y): the reference's tolerance
    (linalg.py:51-54, or the caller's ``tol``), raised to what the compute
    precision resolves."""
    key = _dtype_key(be)
    ref = (max(rows, cols) * np.finfo(np.float64).eps) if tol is None else float(tol)
    return max(ref, RESOLVE[key] * SHIFT_REL[key] ** 0.5)


def _pass2_floor(be, f: float) -> float:
    """Pivot-ratio floor of pass 2 equivalent to the floor f on sigma(Y)."""
    return min(1.0, f / SHIFT_REL[_dtype_key(be)] ** 0.5)


def _svd_rank_basis(be, y, f: float):
    """The reference's rank decision (linalg.py:57-81: keep |R_ii| >= f
    max|R_ii|) on y's singular values from the one-sided Jacobi SVD (eps
    sigma_1 absolute, no squaring); returns the leading left singular vectors."""
    u, sv, _ = be.svd_cols(y)
    k = int((sv > f * sv[0]).sum().item()) if float(sv[0]) > 0 else 0
    if k == 0:
        raise ValueError("cannot orthonormalize an all-zero matrix")
    return be.to_compute(u[:, :k])


def orthonormalize(be, comm, y, tol=None, rows_total: int | None = None, lazy: bool = False,
                   passes: int = 3, planes_out: bool = False):
    """Orthonormal basis of range(y), numerically rank-truncated (linalg.py:57-81),
    by shifted CholeskyQR3 (see SHIFT_REL).

    ``lazy``: no host synchronisation; a rank-deficiency flag (pass 2's pivot
    test) or a failed factorisation is only recorded on the device
    (``be.lazy_failed()``) and the caller must redo the computation eagerly,
    where the truncating eigen path runs.  ``passes=1`` (lazy only): the
    shifted pass alone -- same span, no rank test; used for the
    stabilisations inside the power iteration, whose only job is to keep the
    block well conditioned (the final Q always gets all three passes)."""
    if hasattr(be, "orth_planes") and not isinstance(y, np.ndarray) and hasattr(y, "hi"):
        # y given as the fp16 planes of its transpose (the lazy planes path)
        rows_total = y.cols if rows_total is None else rows_total
        t2 = _pass2_floor(be, rank_floor(be, rows_total, y.rows, tol))
        if lazy and passes == 3:
            return be.orth_planes(comm, y, t2, SHIFT_REL[_dtype_key(be)], planes_out)
        y = be.planes_to_compute(y)
    c = y.shape[1]
    rows_total = y.shape[0] if rows_total is None else rows_total
    key = _dtype_key(be)
    f = rank_floor(be, rows_total, c, tol)
    t2 = _pass2_floor(be, f)
    y_in = y
    # rank deficient in fp64 (eager): the Gram squares y's spectrum, so what
    # the reference's pivoted QR keeps between its floor (max(m, c) eps) and
    # ~sqrt(shift) -- an fp32 input's rounding noise on an exactly low-rank
    # matrix, say -- lies under the shift (or breaks the shifted factor when
    # max G_ii is far below ||G||): decide the rank on y's own singular values
    svd_rank = (not lazy and key == "float64" and hasattr(be, "svd_cols")
                and getattr(comm, "world", 1) == 1 and y.shape[0] >= c)
    g = comm.allreduce_(be.gram64(y))
    x1 = be.chol_inv64(g, 0.0, lazy=lazy, shift=SHIFT_REL[key])
    if passes == 3 and hasattr(be, "save_pivots"):
        be.save_pivots(c)      # Y's pivot range (see CudaBackend.piv)
    if x1 is None and svd_rank:
        return _svd_rank_basis(be, y_in, f)
    if x1 is None:
        # G is indefinite beyond the shift (all-zero or degenerate input):
        # truncate on G's own spectrum, dropping what lies under the shift
        w, v = be.eig_desc64(g)
        t, k = be.eig_orth64(w, v, max(f * f, SHIFT_REL[key]))
        if k == 0:
            raise ValueError("cannot orthonormalize an all-zero matrix")
        y = be.mm(y, be.to_compute(be.cols(t, k)))
        g = comm.allreduce_(be.gram64(y, accurate=True))
        x1 = be.chol_inv64(g, 0.0, shift=SHIFT_REL[key])
        if x1 is None:
            raise RuntimeError("orthonormalize: Cholesky failed after rank truncation")
    q = be.mm(y, be.to_compute(x1), tb=True)
    if lazy and passes == 1:
        return q
    g2 = comm.allreduce_(be.gram64(q, accurate=True))
    x2 = be.chol_inv64(g2, t2, lazy=lazy)
    if x2 is None and svd_rank:
        return _svd_rank_basis(be, y_in, f)
    if x2 is None:
        # rank deficient: keep the directions of q whose pass-2 pivots clear
        # t2 (sigma_i(Y) >= f sigma_1(Y)), as the pivoted QR keeps |R_ii|
        w, v = be.eig_desc64(g2)
        t, k = be.eig_orth64(w, v, t2 * t2)
        if k == 0:
            raise ValueError("cannot orthonormalize an all-zero matrix")
        q = be.mm(q, be.to_compute(be.cols(t, k)))
        g2 = comm.allreduce_(be.gram64(q, accurate=True))
        x2 = be.chol_inv64(g2, 0.0)
        if x2 is None:
            raise RuntimeError("orthonormalize: Cholesky failed after rank truncation")
    q = be.mm(q, be.to_compute(x2), tb=True)
    g3 = comm.allreduce_(be.gram64(q, accurate=True))
    x3 = be.chol_inv64(g3, 0.0, lazy=lazy)
    if x3 is None:
        raise RuntimeError("orthonormalize: third CholeskyQR pass failed")
    return be.mm(q, be.to_compute(x3), tb=True)


def power_iterate(be, comm, atil, omega, q: int, stabilized: bool = True, rows_total=None,
                  lazy: bool = False, gram=None):
    """power.py:113-134 on a row slab of A~: Y = A~ Omega, then q x
    {orth(Y) if stabilized; Z = sum_p A~_p^T Y_p; Y = A~ Z}.  A~ feeds all
    1 + 2q products, so it is prepared once (be.prepare: the fp16 split of
    the 3xFP16 GEMM on the CUDA backend).  gram: G = A~^T A~ already formed
    for the sketch-space path (streamed uploads accumulate it per block)."""
    atil = be.prepare(atil)
    # the power of A~'s spectrum in Y's: 1 for Y = A~ Omega (q = 0), else 2
    # (both paths end with Y = A~ A~^T Q_prev, Q_prev orthonormal) -- read by
    # the fp32 facade's promotion test on Y's pivot range
    be.y_power = 1 if q == 0 else 2
    if lazy and stabilized and q > 0 and hasattr(be, "gram_ok") and be.gram_ok(atil, omega, q):
        return be.power_gram(comm, atil, omega, q, SHIFT_REL[_dtype_key(be)], g=gram)
    if lazy and stabilized and q > 0 and hasattr(be, "planes_ok") and be.planes_ok(atil, omega):
        return be.power_lazy_planes(comm, atil, omega, q, SHIFT_REL[_dtype_key(be)])
    y = be.mm(atil, omega)
    for _ in range(q):
        if stabilized:
            y = orthonormalize(be, comm, y, rows_total=rows_total, lazy=lazy,
                               passes=1 if lazy else 3)
        z = comm.allreduce_(be.mm(atil, y, ta=True))
        y = be.mm(atil, z)
    return y


GRAM_SVD_FLOOR = 1.5e-3   # fp64 randsvd: below it, the SVD of B^T instead of eig(B B^T)


def randsvd(be, comm, a, qb, check: bool = True, amax_hint=None, stats: dict | None = None):
    """power.py:181-199: B = Q^T A (summed over row slabs), thin SVD of B via
    the fp64 Gram B B^T and the eigensolver; U = Q U~, V = B^T U~ / sigma.

    B is formed transposed, B^T = A^T Q (n x c): the long dimension n then
    sits on the GEMM's M side (full 256-row CTA-pair tiles) instead of the
    short c, and B B^T = (B^T)^T B^T, V = B^T U~ read it directly.

    ``check``: the reference's ||Q^T Q - I||_max test (power.py:194-196).  On
    backends with a device-side deviation (``orth_dev_t``) it is queued with
    the rest and read once at the end, with the overflow flag -- no host
    synchronisation between the check and the products.

    ``stats`` (optional dict) receives "qa2", a device scalar with
    ||A||_F^2 - ||A - Q Q^T A||_F^2 = 2 tr(B B^T) - <Q^T Q, B B^T> (exact for
    any Q, so the error identity does not assume Q^T Q = I: with an fp32 Q,
    ||Q^T Q - I|| ~ 1e-6 would otherwise move a small rel_err by ~1e-6 / rel^2)."""
    dev = None
    gq = None
    if check:
        if hasattr(be, "orth_dev_t"):
            gq = comm.allreduce_(be.gram64_q(qb))
            dev = be.orth_dev_t(gq)
        else:
            g = comm.allreduce_(be.gram64(be.dense(qb) if hasattr(be, "dense") else qb))
            _raise_if_not_orthonormal(be, be.orth_dev(g))
    out = _randsvd_core(be, comm, be.mm_at_big(a, qb, amax_hint), qb, gq, stats)
    if dev is not None:
        _raise_if_not_orthonormal(be, be.scalar(dev))
    if be.overflowed(comm):
        # the in-kernel fp16 split met an entry beyond its exponent bound (a
        # hint that did not hold): recompute with 3xTF32 on every rank.  The
        # flag is read once, after everything is queued (no mid-call sync).
        out = _randsvd_core(be, comm, be.mm(a, be.dense(qb), ta=True), qb, gq, stats)
    return out


def _raise_if_not_orthonormal(be, dev: float):
    if not dev <= ORTHO_TOL[_dtype_key(be)]:
        raise ValueError(f"Q is not orthonormal (deviation {dev:.3e})")


def _randsvd_core(be, comm, bt, qb, gq=None, stats=None):
    bt = comm.allreduce_(bt)
    n, c = bt.shape
    world = getattr(comm, "world", 1)
    if world > 1:
        # B B^T = sum over the n rows of B^T: each rank forms the Gram of its
        # 1/world of them and the c x c partial Grams are summed -- the O(n c^2)
        # fp64 Gram is not replicated on every rank (C5 at 8 ranks: 6.3 ->
        # 0.8 ms per rank, SURVEY.md §8(e) strong-scaling limiters)
        r0 = n * comm.rank // world
        r1 = n * (comm.rank + 1) // world
        gb = comm.allreduce_(be.gram64_rows_t(bt[r0:r1]))
    else:
        gb = be.gram64_rows_t(bt)                           # c x c, fp64
    if stats is not None:
        stats["qa2"] = be.proj_sq(gb, gq)
    w, v = be.eig_desc64(gb)
    p = min(c, n)
    sig, inv = be.sqrt_eigs(w)
    planes = hasattr(qb, "hi")          # Q given as the fp16 planes of Q^T
    if (hasattr(be, "svd_cols") and _dtype_key(be) == "float64" and 1 < p == c
            and float(sig[p - 1]) < GRAM_SVD_FLOOR * float(sig[0])):
        # B B^T squares B's condition number: sigma_i below ~1.5e-3 sigma_1
        # would miss the 1e-10 bar (eps (sigma_1 / sigma_i)^2); the one-sided
        # Jacobi SVD of B^T itself keeps eps sigma_1 absolute (the reference's
        # gesdd of B, linalg.py:84-88)
        vb, s, ub = be.svd_cols(bt)     # B^T = Vb S Ub^T: B's left vectors Ub
        u = be.mm(qb, be.to_compute(ub[:, :p]), ta=planes)
        return u, s[:p], be.to_compute(vb[:, :p])
    vc = be.to_compute(be.cols(v, p))
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
