"""GEMM probe: tcgen05 3xTF32 correctness over layouts + timing at C3 shapes."""
import sys, time, json
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops, _lib

lib = _lib.load()
print("tcgen05:", lib.skp_has_tcgen05(), flush=True)
torch.manual_seed(0)
dev = "cuda"

def rnd(r, c, padded):
    if not padded:
        return torch.randn(r, c, device=dev)
    t = _ops.empty2d(r, c, torch.float32, dev)
    t.copy_(torch.randn(r, c, device=dev))
    return t

def check(M, N, K, ta, tb, beta=0.0, padded=False):
    a = rnd(*((K, M) if ta else (M, K)), padded)
    b = rnd(*((N, K) if tb else (K, N)), padded)
    ref = (a.double().T if ta else a.double()) @ (b.double().T if tb else b.double())
    c0 = torch.randn(M, N, device=dev)
    out = c0.clone()
    _ops.gemm(a, b, bool(ta), bool(tb), alpha=1.0, beta=beta, out=out, mode="3xtf32")
    torch.cuda.synchronize()
    exp = ref + beta * c0.double()
    err = ((out.double() - exp).abs().max() / ref.abs().max()).item()
    return err

for (M, N, K) in [(128, 16, 16), (128, 128, 64), (256, 176, 1000), (300, 110, 77), (1000, 520, 4000), (4000, 520, 20000), (67, 45, 131)]:
    for ta in (0, 1):
        for tb in (0, 1):
            try:
                for pad in (False, True):
                    e = check(M, N, K, ta, tb, beta=0.5 if (M + ta) % 2 else 0.0, padded=pad)
                    print(f"M={M} N={N} K={K} ta={ta} tb={tb} pad={int(pad)} relerr={e:.2e}", flush=True)
            except Exception as ex:
                print(f"M={M} N={N} K={K} ta={ta} tb={tb} EXC {ex}", flush=True)

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

res = {}
m, l, r2, n = 262144, 4000, 520, 16384
at = torch.randn(m, l, device=dev)
z = torch.randn(l, r2, device=dev)
y = torch.randn(m, r2, device=dev)
out_nn = torch.empty(m, r2, device=dev)
out_tn = torch.empty(l, r2, device=dev)
for mode in ("3xtf32", "fp32"):
    t = timeit(lambda: _ops.gemm(at, z, out=out_nn, mode=mode))
    f = 2.0 * m * l * r2
    res[f"nn_{mode}"] = (t, f / t / 1e9)
    t = timeit(lambda: _ops.gemm(at, y, True, False, out=out_tn, mode=mode))
    res[f"tn_{mode}"] = (t, f / t / 1e9)
torch.backends.cuda.matmul.allow_tf32 = False
t = timeit(lambda: torch.matmul(at, z, out=out_nn)); res["torch_fp32_nn"] = (t, 2.0 * m * l * r2 / t / 1e9)
torch.backends.cuda.matmul.allow_tf32 = True
t = timeit(lambda: torch.matmul(at, z, out=out_nn)); res["torch_tf32_nn"] = (t, 2.0 * m * l * r2 / t / 1e9)
for k, (t, tf) in res.items():
    print(f"{k:16s} {t:8.3f} ms  {tf:8.1f} TFLOP/s", flush=True)
