"""K2 v2 timing at C3/C5 shapes vs K2 v1."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
from paper_2605_09755_b200.sketching import make_sketch

def timeit(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

SHAPES = [(262144, 16384, 4000), (262144, 16384, 8000), (65536, 24576, 4096)]
if len(sys.argv) > 1:
    SHAPES = SHAPES[:int(sys.argv[1])]
for (m, n, l) in SHAPES:
    a = _ops.empty2d(m, n, torch.float32, "cuda"); a.normal_()
    op = make_sketch("countsketch", n, l, 7, s=8)
    out = _ops.empty2d(m, l, torch.float32, "cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    import time
    plan = op.gather_plan()
    op2 = make_sketch("countsketch", n, l, 8, s=8)
    torch.cuda.synchronize()
    t0 = time.time(); op2.gather_plan(); torch.cuda.synchronize(); tp = time.time() - t0
    gb = (m * n * 4 + m * l * 4) / 1e9
    if plan is not None:
        t2 = timeit(lambda: op.right_permuted(a, out=out, nonfinite=nf))
        print(f"v2 m={m} n={n} l={l}: {t2:.3f} ms  {gb / t2 * 1e3:.1f} GB/s  (plan {tp*1e3:.1f} ms)", flush=True)
    else:
        print(f"v2 m={m} n={n} l={l}: plan unsupported", flush=True)
    t1 = timeit(lambda: op.right(a, out=out, nonfinite=nf), reps=2)
    print(f"v1 m={m} n={n} l={l}: {t1:.3f} ms  {gb / t1 * 1e3:.1f} GB/s", flush=True)
    del a, out
