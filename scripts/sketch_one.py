"""One C3-shape sketch apply (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch
m, n, l = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (262144, 16384, 4000)))
a = torch.randn(m, n, device="cuda")
op = make_sketch("countsketch", n, l, 7, s=8)
out = torch.empty(m, l, device="cuda")
for _ in range(2):
    op.right(a, out=out)
torch.cuda.synchronize()
print("ok")
