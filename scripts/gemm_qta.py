"""Time the C3 Q^T A GEMM (520 x 16384, K = 262144) and the power GEMMs, pair vs 1-CTA."""
import os, sys, subprocess
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
m, n, l, r2 = 262144, 16384, 4000, 520
def mk(r, c):
    t = _ops.empty2d(r, c, torch.float32, "cuda"); t.normal_(); return t
q = mk(m, r2); a = mk(m, n)
out = _ops.empty2d(r2, n, torch.float32, "cuda")
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps
ms = t(lambda: _ops.gemm(q, a, ta=True, out=out, mode="3xtf32"))
print(f"QtA {ms:.3f} ms  {2*m*n*r2/ms/1e9:.1f} TFLOP/s (useful)")
ref = (q[:4096].double().T @ a[:4096, :256].double())
q2 = q[:4096].contiguous(); a2 = a[:4096, :256].contiguous()
o2 = _ops.gemm(_ops.aligned2d(q2) if hasattr(_ops, "aligned2d") else q2, a2, ta=True, mode="3xtf32")
print("check", ((o2.double() - ref).abs().max() / ref.abs().max()).item())
'''
for env in ({}, {"SKP_TC_NO2CTA": "1"}):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(env, r.stdout.strip(), r.stderr[-400:], flush=True)
