"""Dense peaks next to ours (TF32 / FP64 rooflines): cuBLAS
through torch (bf16, TF32, FP64) and this repo's kernels (3xFP16 K4h, 3xTF32
K4, fp64 SIMT K4d) on square N^3 products, CUDA events, best of 5."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops

N = 8192


def best(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return min(t)


flop = 2.0 * N ** 3
g = torch.Generator(device="cuda").manual_seed(0)
rows = []
for name, dt, tf32 in [("cuBLAS bf16", torch.bfloat16, False), ("cuBLAS TF32", torch.float32, True),
                       ("cuBLAS FP32 (no TF32)", torch.float32, False), ("cuBLAS FP64", torch.float64, False)]:
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(N, N, generator=g, device="cuda").to(dt)
    b = torch.randn(N, N, generator=g, device="cuda").to(dt)
    ms = best(lambda: a @ b)
    rows.append((name, ms, flop / ms / 1e9))
torch.backends.cuda.matmul.allow_tf32 = False
a = torch.randn(N, N, generator=g, device="cuda")
b = torch.randn(N, N, generator=g, device="cuda")
sa, sb = _ops.split_h2(a), _ops.split_h2(b, trans=True)
rows.append(("skp K4h 3xFP16 (useful fp32 flop)", best(lambda: _ops.gemm_h3(sa, sb)), None))
rows.append(("skp K4 3xTF32 tcgen05 (useful)", best(lambda: _ops.gemm(a, b, mode="3xtf32")), None))
a64, b64 = a.double(), b.double()
rows.append(("skp K4d fp64 DMMA", best(lambda: _ops.gemm(a64, b64), reps=2), None))
for name, ms, tf in rows:
    tf = flop / ms / 1e9 if tf is None else tf
    print(f"{name:36s} {ms:8.3f} ms  {tf:8.1f} TFLOP/s")
