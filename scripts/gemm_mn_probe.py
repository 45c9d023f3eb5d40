import os, sys, subprocess
variants = ["0,1024,512", "0,512,1024", "1,512,1024", "1,1024,512", "0,1024,1024", "1,512,512"]
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
torch.manual_seed(0)
for (M, N, K) in [(128, 16, 16), (256, 176, 1000)]:
    for ta, tb in [(1, 1), (0, 0), (1, 0)]:
        a = torch.randn((K, M) if ta else (M, K), device="cuda")
        b = torch.randn((N, K) if tb else (K, N), device="cuda")
        ref = (a.double().T if ta else a.double()) @ (b.double().T if tb else b.double())
        out = _ops.gemm(a, b, bool(ta), bool(tb), mode="3xtf32")
        torch.cuda.synchronize()
        err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
        print(f"  M={M} N={N} K={K} ta={ta} tb={tb} relerr={err:.2e} maxout={out.abs().max().item():.3e}", flush=True)
'''
for v in variants:
    print("variant", v, flush=True)
    env = dict(os.environ, SKP_TC_MN=v)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    print(r.stdout[-2000:], r.stderr[-500:], flush=True)
