"""randsvd on an unaligned-row device A (n = 4001, the pre-fix upload) vs the
padded copy the upload now makes, both against the oracle's sigma."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import datagen, power, _ops
from oracle import skp_oracle as o
m, l, r2, k = 65536, 600, 80, 60
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4001
a = datagen.lowrank_plus_noise_gpu(m, n, np.exp(-np.arange(1.0, 513.0) / 60.0), 1e-8, seed=9).cpu().numpy()
spec = skp.RangeFinderSpec(k=k, l=l, r1=l, r2=r2, q=2, eps=0.5, seed=9, s=8)
qb = skp.range_finder_sketched(torch.from_numpy(a).cuda(), spec)   # CUDA in -> CUDA out
qo = o.range_finder_sketched(a, o.Spec(k=k, l=l, r1=l, r2=r2, q=2, seed=9, s=8))
_, so, _ = o.randsvd(a, qo)
t_unal = torch.from_numpy(a).cuda()                                 # stride 4001 (unaligned)
t_pad = _ops.empty2d(m, n, torch.float32, "cuda"); t_pad.copy_(t_unal)
for name, t in (("unaligned rows (pre-fix upload)", t_unal), ("128-byte rows (upload now)", t_pad)):
    power._randsvd_dev(t, qb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, s, _ = power._randsvd_dev(t, qb)
    e1.record()
    torch.cuda.synchronize()
    err = np.abs(s.cpu().numpy()[:k] - so[:k]) / so[:k]
    print(f"n={n} {name}: max rel sigma diff {err.max():.2e}, randsvd {e0.elapsed_time(e1):.2f} ms")
