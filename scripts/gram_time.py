"""The CholeskyQR Gram (K-major SYRK of Y^T's planes) at (N, K): python scripts/gram_time.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
for n, k in ((1050, 1 << 20), (520, 262144), (1050, 131072), (2048, 1 << 18)):
    y = _ops.empty2d(k, n, torch.float32, "cuda")
    y.normal_()
    yt = _ops.split_h2(y, trans=True)
    for _ in range(2):
        g = _ops.syrk_h3(yt, rows=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g = _ops.syrk_h3(yt, rows=True)
    e1.record()
    torch.cuda.synchronize()
    ref = (y.double().T @ y.double())
    err = ((g.double() - ref).abs().max() / ref.abs().max()).item()
    print(f"N={n} K={k}: {e0.elapsed_time(e1) / 5:.3f} ms  max rel err {err:.2e}", flush=True)
    del y, yt, g, ref
    torch.cuda.empty_cache()
