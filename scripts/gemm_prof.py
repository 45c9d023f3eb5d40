"""Run the C3-shaped NN GEMM once under SKP_TC_PROF with several debug modes."""
import os, sys, subprocess
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
m, l, r2 = 262144, 4000, 520
at = _ops.empty2d(m, l, torch.float32, "cuda"); at.normal_()
z = _ops.empty2d(l, r2, torch.float32, "cuda"); z.normal_()
out = _ops.empty2d(m, r2, torch.float32, "cuda")
_ops.gemm(at, z, out=out, mode="3xtf32"); torch.cuda.synchronize()
'''
modes = [{}]
for env in modes:
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SKP_TC_PROF="1", **env),
                       capture_output=True, text=True)
    print(env, "\n" + r.stderr.strip()[-900:], flush=True)
