"""K2 v2 timing at C3 (alone, CUDA events) and the plan build time."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch
m, n, l = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (262144, 16384, 4000)))
a = torch.randn(m, n, device="cuda")
out = torch.empty(m, l, device="cuda")
nonfinite = torch.zeros(1, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for seed in (7, 8):
    op = make_sketch("countsketch", n, l, seed, s=8)
    torch.cuda.synchronize()
    e0.record()
    op.gather_plan(check=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"seed {seed}: plan {e0.elapsed_time(e1):.3f} ms")
for _ in range(2):
    op.right_permuted(a, out=out, nonfinite=nonfinite)
e0.record()
for _ in range(5):
    op.right_permuted(a, out=out, nonfinite=nonfinite)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"K2 v2 {m}x{n}->{l}: {ms:.3f} ms  {(m * n * 4 + m * l * 4) / ms / 1e6:.0f} GB/s  nonfinite {int(nonfinite.item())}")
