"""K2 v2 plan quality: LDS steps (sum over warps of T), shared-memory
wavefronts (max distinct words per bank per step) and the ideal
(entries / 32), per column pass.   python scripts/plan_stats.py n l"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch, substream
n, l = int(sys.argv[1]), int(sys.argv[2])
op = make_sketch("countsketch", n, l, substream(3, 0), s=8, device="cuda")
plan, _ = op.gather_plan()
H = -(-n // (24608 - 32))
npass = -(-(-(-n // H)) // 32) * 32
V = 1                                           # sketch_gather.cu: one column per lane
W = 20 if V == 2 else 28
COLS, TMAX = 32 * W * V, 128
SPARE = COLS * 3 // 28
P = -(-l // (COLS - SPARE))
g = plan.cpu().numpy().view(np.uint32)
o = (P * COLS * 4 + 15) // 16 * 16 // 4 + 4   # perm, fail (16 B)
entries = n * 8
tot_steps = tot_wf = 0
for h in range(H):
    VW = W * V
    tw = g[o:o + P * VW].astype(np.int64)
    o += (P * VW * 4 + 15) // 16 * 16 // 4
    sched = g[o:o + P * VW * TMAX * 32].reshape(P * VW, TMAX, 32)
    o += P * VW * TMAX * 32
    steps = int(tw.sum())
    wf = 0
    for w in range(P * VW):
        t = tw[w]
        if t == 0:
            continue
        words = (sched[w, :t] & 0x7fffffff) >> 2
        banks = words & 31
        for tt in range(t):
            wb, bb = words[tt], banks[tt]
            cnt = np.zeros(32, np.int64)
            for b in np.unique(bb):
                cnt[b] = len(np.unique(wb[bb == b]))
            wf += cnt.max()
    tot_steps += steps
    tot_wf += wf
    print(f"pass {h}: V={V} virtual warps {P * VW} steps {steps} (mean T {steps / max(1, (tw > 0).sum()):.1f}, max {tw.max()}) wavefronts {wf} ({wf / steps:.3f} per LDS)")
ideal = entries / 32
print(f"total: steps {tot_steps} wavefronts {tot_wf}; ideal {ideal:.0f} -> padding x{tot_steps / ideal:.3f}, "
      f"conflicts x{tot_wf / tot_steps:.3f}, overall x{tot_wf / ideal:.3f}; P={P} slices, H={H} passes; "
      f"ingest {P * H * n / 32 / H:.0f} wavefronts per row vs gather {tot_wf:.0f}/row")
