"""Per-stage cost of the tcgen05 GEMM pipeline under debug knobs (layouts x N)."""
import os, sys, subprocess
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
m, K = 65536, 4000
def mk(r, c):
    t = _ops.empty2d(r, c, torch.float32, "cuda"); t.normal_(); return t
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps
out = []
for N in (128, 256, 520):
    tn = -(-N // 256); bn = -(-(-(-N // tn)) // 16) * 16
    stages_per_sm = (m // 128) * tn / 148 * (K // 16)
    for ta in (0, 1):
        for tb in (0, 1):
            a = mk(K, m) if ta else mk(m, K)
            b = mk(N, K) if tb else mk(K, N)
            c = mk(m, N)
            ms = t(lambda: _ops.gemm(a, b, bool(ta), bool(tb), out=c, mode="3xtf32"))
            cyc = ms * 1e-3 * 1.9e9 / stages_per_sm
            out.append(f"N={N} bn={bn} ta={ta} tb={tb}: {ms:.3f} ms  {cyc:.0f} cyc/stage")
print("\n".join(out))
'''
for env in ({"SKP_TC_DBG": "8", "SKP_TC_RAW1": "1"}, {"SKP_TC_DBG": "8"}, {"SKP_TC_DBG": "12"}, {}):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(env, "\n" + r.stdout.strip(), r.stderr[-300:], flush=True)
