import sys, numpy as np
sys.path.insert(0, ".")
from oracle import skp_oracle as o
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import datagen
m, n = 4000, 1000
a = datagen.rotate_spectrum(m, n, max(m, n) / np.arange(1.0, n + 1.0), 11).astype(np.float32)
for q in (0, 1, 2):
    ospec = o.Spec(k=100, l=300, r1=300, r2=120, q=q, seed=5, s=8)
    qo = o.range_finder_sketched(a, ospec)
    _, so, _ = o.randsvd(a, qo)
    spec = skp.RangeFinderSpec(k=100, l=300, r1=300, r2=120, q=q, eps=0.5, seed=5, s=8)
    qb = skp.range_finder_sketched(a, spec).astype(np.float64)
    dev = np.abs(qb.T @ qb - np.eye(qb.shape[1])).max()
    s_np = np.linalg.svd(qb.T @ a.astype(np.float64), compute_uv=False)
    res = skp.randsvd(a, qb.astype(np.float32))
    print(q, qb.shape, "orth dev %.2e" % dev, "sig(np) rel %.2e" % np.abs(s_np[:100] / so[:100] - 1).max(),
          "sig(randsvd) rel %.2e" % np.abs(res.sigma[:100] / so[:100] - 1).max(), flush=True)
    r2, rel = skp.rsvd(a, spec, with_error=True)
    print("   rsvd sig rel %.2e" % np.abs(np.asarray(r2.sigma[:100]) / so[:100] - 1).max(), "rel", rel, o.proj_rel_error(a, qo))
    import torch
    from paper_2605_09755_b200 import power
    qd = power._range_finder_dev(torch.from_numpy(a).cuda(), spec, planes_out=True)
    qd = qd.double().cpu().numpy()
    print("   dev Q orth %.2e" % np.abs(qd.T @ qd - np.eye(qd.shape[1])).max(), qd.shape)
