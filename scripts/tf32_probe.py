"""Does tcgen05 kind::tf32 truncate or round raw fp32 operands?"""
import os, sys, subprocess
code = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
torch.manual_seed(1)
M, N, K = 256, 128, 512
a = torch.randn(M, K, device="cuda"); b = torch.randn(K, N, device="cuda")
def trunc(x): return (x.view(torch.int32) & -8192).view(torch.float32)
def rnd(x): return ((x.view(torch.int32) + 4096) & -8192).view(torch.float32)
out = _ops.gemm(a, b, mode="3xtf32")
ref_t = trunc(a).double() @ trunc(b).double()
ref_r = rnd(a).double() @ rnd(b).double()
ref = a.double() @ b.double()
print("vs trunc", (out.double() - ref_t).abs().max().item(), "vs round", (out.double() - ref_r).abs().max().item(), "vs exact", (out.double()-ref).abs().max().item())
'''
env = dict(os.environ, SKP_TC_RAW1="1")
r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
print("raw1:", r.stdout, r.stderr[-300:])
r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
print("3x:", r.stdout, r.stderr[-300:])
