import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from test_gpu_sweep import _case, _matrix
import paper_2605_09755_b200 as skp
from oracle import skp_oracle as o
i = 8
m, n, l, r2, k, q, s, dtype, cuda_in, rank, decay = _case(i)
a = _matrix(m, n, rank, decay, i, dtype)
spec = skp.RangeFinderSpec(k=k, l=l, r1=l, r2=r2, q=q, eps=0.5, seed=i, s=s)
qo = o.range_finder_sketched(a, o.Spec(k=k, l=l, r1=l, r2=r2, q=q, seed=i, s=s))
print("oracle cols", qo.shape[1], "orth", np.abs(qo.T @ qo - np.eye(qo.shape[1])).max())
for dt in (np.float64, np.float32):
    qb = skp.range_finder_sketched(a.astype(dt), spec)
    print(dt.__name__, "cols", qb.shape[1], qb.dtype, "orth", np.abs(qb.T.astype(np.float64) @ qb - np.eye(qb.shape[1])).max())
