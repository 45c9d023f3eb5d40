"""apply_right's device op (SketchOperator.right) at a C5 row slab: K2 v2 +
un-permutation against K2 v1.   python scripts/right_time.py [m n l]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
from paper_2605_09755_b200.sketching import make_sketch
m, n, l = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (131072, 32768, 8000)))
a = _ops.empty2d(m, n, torch.float32, "cuda")
a.normal_()
op = make_sketch("countsketch", n, l, 7, s=8)
out = _ops.empty2d(m, l, torch.float32, "cuda")


def t(f, k=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


ms2 = t(lambda: op.right(a, out=out))
ref = out.clone()
ms1 = t(lambda: _ops.sketch_right(a, op.colptr, op.entries, op.s, op.r, out))
diff = (ref - out).abs().max().item()
ms_g = t(lambda: op.right_permuted(a, out=out))
ms_u = t(lambda: _ops.unpermute_cols(out, op.right_permuted(a, out=out)[1]), 3) - ms_g
print(f"m={m} n={n} l={l}: right (v2 + unpermute) {ms2:.2f} ms, v1 {ms1:.2f} ms, "
      f"v2 gather alone {ms_g:.2f} ms, unpermute ~{ms_u:.2f} ms; max|v2 - v1| "
      f"{diff:.3e} (scale {ref.abs().max().item():.3e})")
