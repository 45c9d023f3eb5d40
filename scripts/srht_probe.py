"""K7 SRHT apply at the C3 shape (A 262144 x 16384, r = 4000)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
from paper_2605_09755_b200.sketching import make_sketch
m, n, r = 262144, 16384, 4000
a = _ops.empty2d(m, n, torch.float32, "cuda"); a.normal_()
op = make_sketch("srht", n, r, 7)
out = _ops.empty2d(m, r, torch.float32, "cuda")
op.right(a, out=out); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3):
    op.right(a, out=out)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 3
print(f"srht A S {m}x{n} -> r={r}: {t:.3f} ms  {(m * n * 4 + m * r * 4) / t / 1e6:.0f} GB/s")
