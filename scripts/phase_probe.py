"""Phase times of the C3 rSVD step, back to back vs with an idle gap before each step."""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import datagen, distributed as D
m, n = 262144, 16384
a = datagen.c3_matrix_gpu(3, m, n, device="cuda")
spec = skp.RangeFinderSpec(k=500, l=4000, r1=4000, r2=520, q=3, eps=0.5, s=8, seed=3)
class L:
    rank, world = 0, 1
    def allreduce_(self, t): return t
for gap in (0.0, 0.2, 0.0):
    for _ in range(2):
        D.rsvd_sharded(a, spec, m, L(), None, with_error=False)
    torch.cuda.synchronize()
    ph = {}
    for _ in range(4):
        if gap:
            torch.cuda.synchronize(); time.sleep(gap)
        D.rsvd_sharded(a, spec, m, L(), ph, with_error=False)
    print(f"gap {gap}: " + " ".join(f"{k} {v / 4:.2f}" for k, v in ph.items()), flush=True)
