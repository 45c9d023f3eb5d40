import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from test_gpu_sweep import _case, _matrix
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import power, _engine
from oracle import skp_oracle as o
i = int(sys.argv[1]) if len(sys.argv) > 1 else 6
m, n, l, r2, k, q, s, dtype, cuda_in, rank, decay = _case(i)
a = _matrix(m, n, rank, decay, i, dtype)
spec = skp.RangeFinderSpec(k=k, l=l, r1=l, r2=r2, q=q, eps=0.5, seed=i, s=s)
qo = o.range_finder_sketched(a, o.Spec(k=k, l=l, r1=l, r2=r2, q=q, seed=i, s=s))
_, so, _ = o.randsvd(a, qo)
hint = {}
t = torch.from_numpy(a).cuda()
qd = power._range_finder_dev(t, spec, hint_out=hint)
qb = qd.cpu().numpy()
print("cols", qb.shape[1], qo.shape[1], "pivot_ratio", hint.get("pivot_ratio"))
s_np = np.linalg.svd(qb.T @ a, compute_uv=False)
print("numpy sigma of our Q^T A vs oracle: max rel", np.max(np.abs(s_np[:k] - so[:k]) / so[:k]))
res = skp.randsvd(a, qb)
print("our randsvd on our Q vs numpy on our Q: max rel", np.max(np.abs(res.sigma[:k] - s_np[:k]) / s_np[:k]))
res2 = skp.randsvd(a, qo)
print("our randsvd on the oracle's Q vs oracle: max rel", np.max(np.abs(res2.sigma[:k] - so[:k]) / so[:k]))
d = np.linalg.norm(qb @ (qb.T @ qo) - qo, 2)
print("subspace distance", d)
