import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2605_09755_b200 as skp
from oracle import skp_oracle as o
for (n, r, s, seed) in [(513, 64, 1, 13), (513, 64, 1, 21), (512, 64, 1, 13), (514, 64, 1, 13), (515, 64, 1, 13), (1025, 64, 1, 13), (513, 200, 1, 13), (513, 64, 1, 5)]:
    op = skp.make_sketch("countsketch", n, r, seed=seed, s=s)
    oc = o.CountSketch("countsketch", n, r, seed, s=s)
    sd = op._signs.reshape(n, s); so = np.asarray(oc.signs).reshape(n, s)
    bad = np.nonzero((sd != so).any(axis=1))[0]
    print((n, r, s, seed), "sign mismatches:", len(bad), bad[:8])
