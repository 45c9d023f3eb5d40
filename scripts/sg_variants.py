import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
from paper_2605_09755_b200.sketching import make_sketch
m, n, l = 262144, 16384, 4000
a = _ops.empty2d(m, n, torch.float32, "cuda"); a.normal_()
op = make_sketch("countsketch", n, l, 7, s=8)
out = _ops.empty2d(m, l, torch.float32, "cuda")
nf = torch.zeros(1, dtype=torch.int64, device="cuda")
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps
print("norms %.3f ms  no-norms %.3f ms" % (t(lambda: op.right_permuted(a, out=out, nonfinite=nf)), t(lambda: op.right_permuted(a, out=out))))
'''
for env in ({}, {"SKP_SG_PF": "0"}, {"SKP_SG_NBUF2": "1", "SKP_SG_PF": "0"}, {"SKP_SG_NBUF2": "1"}, {"SKP_SG_PF": "8"}):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(env, r.stdout.strip(), r.stderr[-300:], flush=True)
