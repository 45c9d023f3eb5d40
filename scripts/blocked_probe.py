import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import datagen, power
m, n, l, r2, k, q, rank = 16384, 4096, 1000, 120, 100, 3, 2048
spec_v = np.arange(1.0, rank + 1.0) ** -0.5
a_dev = datagen.lowrank_plus_noise_gpu(m, n, spec_v, 1e-6, seed=3)
spec = skp.RangeFinderSpec(k=k, l=l, r1=l, r2=r2, q=q, eps=0.5, seed=3, s=8)
for blocked in (False, True):
    if blocked:
        power._atil_blocked = lambda *x: True
        power._BLOCK_BYTES = 1000 * l * 4
    hint = {}
    qb = power._range_finder_dev(a_dev, spec, hint_out=hint)
    print("blocked", blocked, "cols", qb.shape, "pivot_ratio", hint.get("pivot_ratio"))
