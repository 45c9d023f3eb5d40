"""One C3-shape sketch apply (for ncu): python scripts/sketch_one.py [v2|v1] [m n l]

v2 = the row-gather kernel the range finder runs (permuted output columns),
v1 = the rows-in-lanes ELL kernel (fallback)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch
mode = sys.argv[1] if len(sys.argv) > 1 else "v2"
m, n, l = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (262144, 16384, 4000)))
a = torch.empty(m, n, device="cuda")
a.normal_()
op = make_sketch("countsketch", n, l, 7, s=8)
out = torch.empty(m, l, device="cuda")
nonfinite = torch.zeros(1, dtype=torch.int64, device="cuda")
def run():
    if mode == "v2":
        assert op.right_permuted(a, out=out, nonfinite=nonfinite) is not None
    else:
        op.right(a, out=out, nonfinite=nonfinite)


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print("ok", mode, m, n, l, "%.3f ms  %.1f GB/s" % (ms, (m * n * 4 + m * l * 4) / ms / 1e6))
