"""K2 v2 schedule: shared-memory wavefronts per LDS implied by the plan (C3).

For each (warp, step) the 32 lanes read word addresses sched & 0x7fffffff / 4;
wavefronts = max over banks of the distinct words in that bank.  Compares the
plan's ideal (1.0) with what ncu reports for the kernel."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch
n, l = 16384, 4000
op = make_sketch("countsketch", n, l, 7, s=8)
plan, perm = op.gather_plan()
GATHER_COLS = 896  # sketch_gather.cu kGCols
W = GATHER_COLS // 32
P = -(-l // (GATHER_COLS - 96))
g = plan.cpu().numpy().view(np.uint32)
o = P * GATHER_COLS + 4
tw = g[o:o + P * W].astype(np.int64)
o += (P * W + 3) // 4 * 4
sched = g[o:o + P * W * 128 * 32].reshape(P * W, 128, 32)
tot_w = tot_i = 0
hist = np.zeros(40, np.int64)
for w in range(P * W):
    for t in range(tw[w]):
        words = (sched[w, t] & 0x7fffffff) >> 2
        banks = words & 31
        wf = 0
        for b in np.unique(banks):
            wf = max(wf, len(np.unique(words[banks == b])))
        hist[wf] += 1
        tot_w += wf
        tot_i += 1
print("steps", tot_i, "wavefronts", tot_w, "per LDS %.3f" % (tot_w / tot_i))
print("histogram", {i: int(h) for i, h in enumerate(hist) if h})
print("T per warp: mean %.1f max %d" % (tw[tw > 0].mean(), tw.max()))
