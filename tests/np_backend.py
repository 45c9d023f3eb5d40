"""numpy compute backend for the engine -- TEST ONLY.

Implements the ``_engine`` backend interface with numpy/scipy so the
row-sharded orchestration (what is all-reduced, when, in which order) can be
exercised by multi-process gloo tests on a CPU-only box.  The product uses
``_ops.CudaBackend``; nothing in the package imports this module.
"""
import numpy as np


class NumpyBackend:
    name = "numpy"

    def __init__(self, dtype=np.float64):
        self.dtype = np.dtype(dtype)

    def prepare(self, x):
        return x

    def dense(self, q):
        return q

    def mm_at_big(self, a, q, amax_hint=None):
        return self.mm(a, q, ta=True)

    def overflowed(self, comm=None):
        return False

    def mm(self, a, b, ta=False, tb=False, out=None, alpha=1.0, beta=0.0):
        r = (a.T if ta else a) @ (b.T if tb else b)
        return np.ascontiguousarray(r.astype(self.dtype, copy=False))

    def gram64(self, y, accurate=False):
        return np.ascontiguousarray((y.T @ y).astype(np.float64))

    def gram64_rows(self, b):
        b = b.astype(np.float64)
        return b @ b.T

    def gram64_rows_t(self, bt):
        bt = bt.astype(np.float64)
        return bt.T @ bt

    def chol_inv64(self, g, rel_tol, lazy=False, shift=0.0):
        try:
            lmat = np.linalg.cholesky(g + shift * max(float(np.diag(g).max()), 0.0) * np.eye(len(g)))
            d = np.abs(np.diag(lmat))
            ok = d.min() >= rel_tol * d.max()
        except np.linalg.LinAlgError:
            lmat, ok = None, False
        if not ok:
            if lazy:
                self._fail = True
                return np.eye(g.shape[0])
            return None
        return np.linalg.inv(lmat)

    def eig_desc64(self, g):
        w, v = np.linalg.eigh((g + g.T) / 2)
        idx = np.argsort(-w, kind="stable")
        return w[idx], np.ascontiguousarray(v[:, idx])

    def eig_orth64(self, w, v, rel_tol):
        keep = (w > 0) & (w > rel_tol * w[0])
        t = np.zeros_like(v)
        t[:, keep] = v[:, keep] / np.sqrt(w[keep])
        return t, int(keep.sum())

    def sqrt_eigs(self, w):
        s = np.sqrt(np.maximum(w, 0))
        inv = np.where(s > 0, 1 / np.where(s > 0, s, 1), 0)
        return s, inv

    def proj_sq(self, gb, gq=None):
        t = float(np.trace(gb))
        return t if gq is None else 2.0 * t - float((gq * gb).sum())

    def orth_dev(self, g):
        return float(np.abs(g - np.eye(g.shape[0])).max())

    def to_compute(self, x):
        return np.ascontiguousarray(x.astype(self.dtype))

    def scale_cols_(self, x, s):
        x *= s.astype(x.dtype)
        return x

    def symmetrize_(self, w):
        w[...] = (w + w.T) / 2
        return w

    def cols(self, x, k):
        return np.ascontiguousarray(x[:, :k])

    def sumsq(self, x):
        return np.array([float((x.astype(np.float64) ** 2).sum())])

    def scalar(self, x):
        return float(np.asarray(x).reshape(-1)[0])

    # lazy (sync-free) protocol of the CUDA backend: numpy never defers
    def lazy_reset(self):
        self._fail = False

    def lazy_failed(self, comm=None):
        return getattr(self, "_fail", False)
