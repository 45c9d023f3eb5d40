import os, sys, subprocess
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
m, l, r2 = 262144, 4000, 520
at = _ops.empty2d(m, l, torch.float32, "cuda"); at.normal_()
z = _ops.empty2d(l, r2, torch.float32, "cuda"); z.normal_()
y = _ops.empty2d(m, r2, torch.float32, "cuda"); y.normal_()
out = _ops.empty2d(m, r2, torch.float32, "cuda")
outt = _ops.empty2d(l, r2, torch.float32, "cuda")
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps
ms = t(lambda: _ops.gemm(at, z, out=out, mode="3xtf32"))
print(f"NN {ms:.3f} ms  {2*m*l*r2/ms/1e9:.1f} TFLOP/s (useful)")
ms = t(lambda: _ops.gemm(at, y, out=outt, ta=True, mode="3xtf32"))
print(f"TN {ms:.3f} ms  {2*m*l*r2/ms/1e9:.1f} TFLOP/s (useful)")
'''
envs = [{}, {"SKP_TC_FORCE2CTA": "1"}, {"SKP_TC_RAW1": "1"}, {"SKP_TC_NO2CTA": "1"}]
for extra in sys.argv[1:]:
    k, v = extra.split("=")
    envs.append({k: v})
for env in envs:
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(env, r.stdout.strip(), r.stderr[-300:])
