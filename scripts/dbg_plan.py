import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops, _lib
from paper_2605_09755_b200.sketching import make_sketch, substream
n, l = int(sys.argv[1]), int(sys.argv[2])
sk = make_sketch("countsketch", n, l, substream(4, 0), s=8, device="cuda")
counts = np.bincount(sk.d_cols.cpu().numpy().ravel(), minlength=l)
print("entries per column: mean %.1f max %d min %d" % (counts.mean(), counts.max(), counts.min()))
g = _ops.gather_plan(sk.colptr, sk.entries, n, l, "cuda", check=False)
plan = g[0]
off = int(_lib.load().skp_sketch_gather_plan_fail_offset(l))
torch.cuda.synchronize()
print("fail word", int(plan[off:off + 4].view(torch.int32).item()))
