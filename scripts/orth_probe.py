import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from test_gpu_sweep_api import _graded
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import _engine, _ops, linalg
from oracle import skp_oracle as o
rng = np.random.default_rng(2002)
m, c = int(rng.integers(50, 3000)), int(rng.integers(1, 120)); c = min(c, m)
rank = int(rng.integers(1, c + 1)); dtype = np.float32
decades = float(rng.uniform(0, 6))
y = _graded(m, c, decades, rank, 2, dtype)
print(m, c, rank, decades)
print("numpy svd of y (fp64):", np.linalg.svd(y.astype(np.float64), compute_uv=False)[[0, rank - 1, rank, -1]])
print("oracle cols", o.orthonormalize(y).shape[1])
t = torch.from_numpy(y.astype(np.float64)).cuda()
be = linalg._backend(_ops.F64, t.device)
print("backend", type(be).__name__)
q = _engine.orthonormalize(be, _engine.LOCAL, t)
print("fp64 engine cols", q.shape[1])
print("facade fp32 cols", skp.orthonormalize(y).shape[1])
orig_chol = be.chol_inv64
def chol(g, rel_tol, lazy=False, shift=0.0):
    x = orig_chol(g, rel_tol, lazy=lazy, shift=shift)
    print("chol_inv64 n", g.shape[0], "rel_tol", rel_tol, "shift", shift, "->", None if x is None else "ok", "info", be.info.tolist())
    return x
be.chol_inv64 = chol
orig_eo = be.eig_orth64
def eo(w, v, tol):
    t, k = orig_eo(w, v, tol)
    print("eig_orth64 tol", tol, "k", k, "w[0], w[-1]", float(w[0]), float(w[-1]))
    return t, k
be.eig_orth64 = eo
q = _engine.orthonormalize(be, _engine.LOCAL, t)
print("cols", q.shape[1])
