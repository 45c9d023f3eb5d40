"""One C3-shape GEMM (for ncu): python scripts/gemm_one.py nn|tn [3xtf32|h3] [reps]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
kind = sys.argv[1] if len(sys.argv) > 1 else "nn"
mode = sys.argv[2] if len(sys.argv) > 2 else "3xtf32"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
m, l, r2 = 262144, 4000, 520
torch.manual_seed(0)
at = _ops.empty2d(m, l, torch.float32, "cuda")
at.normal_()
if kind == "nn":
    z = _ops.empty2d(l, r2, torch.float32, "cuda")
    z.normal_()
    if mode == "h3":
        sa, sz = _ops.split_h2(at), _ops.split_h2(z, trans=True)
        f = lambda: _ops.gemm_h3(sa, sz)
    else:
        f = lambda: _ops.gemm(at, z, mode=mode)
else:
    y = _ops.empty2d(m, r2, torch.float32, "cuda")
    y.normal_()
    if mode == "h3":
        sa, sy = _ops.split_h2(at), _ops.split_h2(y, trans=True)
        f = lambda: _ops.gemm_h3(sa, sy, ta=True)
    else:
        f = lambda: _ops.gemm(at, y, True, False, mode=mode)
for _ in range(reps):
    f()
torch.cuda.synchronize()
print("ok")
