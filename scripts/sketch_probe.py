"""Sketch K2 probe: correctness vs numpy at small shapes, timing at C3/C4/C5 shapes."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200.sketching import make_sketch

def check(m, n, r, s, dtype):
    rng = np.random.default_rng(m)
    a = rng.standard_normal((m, n)).astype(dtype)
    op = make_sketch("countsketch", n, r, 5, s=s)
    out = op.apply_right(a)
    cols, signs = op._cols, op._signs
    ref = np.zeros((m, r))
    a64 = a.astype(np.float64)
    for t in range(s):
        np.add.at(ref.T, cols[:, t], (a64 * (signs[:, t] / np.sqrt(s))).T)
    return np.abs(out - ref).max() / np.abs(ref).max()

for (m, n, r, s, dt) in [(64, 1000, 200, 8, np.float32), (100, 3000, 1500, 8, np.float32), (33, 700, 4000, 8, np.float32),
                         (257, 2048, 1024, 3, np.float64), (1, 100, 10, 2, np.float32), (70, 1030, 130, 8, np.float64)]:
    print(f"m={m} n={n} r={r} s={s} {dt.__name__} relerr={check(m, n, r, s, dt):.2e}", flush=True)

def timeit(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for (m, n, l) in [(262144, 16384, 4000), (65536, 65536, 4096), (262144, 32768, 8000)]:
    a = torch.randn(m, n, device="cuda")
    op = make_sketch("countsketch", n, l, 7, s=8)
    out = torch.empty(m, l, device="cuda")
    t = timeit(lambda: op.right(a, out=out))
    gb = (m * n * 4 + m * l * 4) / 1e9
    print(f"sketch m={m} n={n} l={l}: {t:.3f} ms  {gb / t * 1e3:.1f} GB/s", flush=True)
    del a, out
    torch.cuda.empty_cache()
