"""K2 v2 plan balance at C3: schedule steps per warp (T) per slice."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch
n, l = 16384, 4000
op = make_sketch("countsketch", n, l, 7, s=8)
plan, perm = op.gather_plan()
P = -(-l // 768)
g = plan.cpu().numpy().view(np.int32)
tw = g[P * 768: P * 768 + P * 24].reshape(P, 24)
cnt = np.diff(op.colptr.cpu().numpy())
print("column counts: mean %.1f min %d max %d" % (cnt.mean(), cnt.min(), cnt.max()))
for p in range(P):
    t = tw[p][tw[p] > 0]
    print(f"slice {p}: warps {len(t)} T max {t.max()} mean {t.mean():.1f} min {t.min()}  efficiency {t.mean() / t.max():.2f}")
