"""One C3-shape GEMM (for ncu): python scripts/gemm_one.py nn|tn [mode] [reps]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
kind = sys.argv[1] if len(sys.argv) > 1 else "nn"
mode = sys.argv[2] if len(sys.argv) > 2 else "3xtf32"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
m, l, r2 = 262144, 4000, 520
torch.manual_seed(0)
at = torch.randn(m, l, device="cuda")
if kind == "nn":
    z = torch.randn(l, r2, device="cuda")
    f = lambda: _ops.gemm(at, z, mode=mode)
else:
    y = torch.randn(m, r2, device="cuda")
    f = lambda: _ops.gemm(at, y, True, False, mode=mode)
for _ in range(reps):
    f()
torch.cuda.synchronize()
print("ok")
