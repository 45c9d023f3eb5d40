"""One config-shape GEMM (for ncu):
    python scripts/gemm_one.py nn|tn|qta|syrk [3xtf32|h3|h3s] [reps] [C3|C5]
(qta: randsvd's B^T = A^T Q with A m x n)"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
kind = sys.argv[1] if len(sys.argv) > 1 else "nn"
mode = sys.argv[2] if len(sys.argv) > 2 else "3xtf32"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = sys.argv[4] if len(sys.argv) > 4 else "C3"
m, n, l, r2 = {"C3": (262144, 16384, 4000, 520), "C5": (1048576, 32768, 8000, 1050)}[cfg]
torch.manual_seed(0)
at = _ops.empty2d(m, l, torch.float32, "cuda")
at.normal_()
if kind == "qta":
    del at
    a = _ops.empty2d(m, n, torch.float32, "cuda")
    a.normal_()
    q = _ops.empty2d(m, r2, torch.float32, "cuda")
    q.normal_()
    if mode == "h3s":
        e_a, sq = _ops.h2_exponent(a), _ops.split_h2(q, trans=True)
        f = lambda: _ops.gemm_h3s_t(a, e_a, sq)
    else:
        f = lambda: _ops.gemm(a, q, True, False, mode=mode)
elif kind == "syrk":
    sa = _ops.split_h2_inplace(at)
    f = lambda: _ops.syrk_h3(sa)
elif kind == "nn":
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
f()
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(reps):
    f()
t1.record()
torch.cuda.synchronize()
print("ok", kind, mode, cfg, "ms per call %.3f" % (t0.elapsed_time(t1) / reps))
