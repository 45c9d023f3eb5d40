"""Tensor-core fp32 accumulation bias: a^T q with a = 1, q = c (K = 262144)
for several split-K chain lengths (SKP_H3_MAXCHAIN), 3xFP16-s and 3xTF32."""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for chain, chunk in ((262144, 8), (262144, 1), (262144, 4096)):
        env = dict(os.environ, SKP_H3_MAXCHAIN=str(chain), SKP_H3_CHUNK=str(chunk))
        print(subprocess.run([sys.executable, __file__, "x"], env=env, capture_output=True,
                             text=True).stdout.strip(), flush=True)
    sys.exit(0)
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
K, M, N = 262144, 256, 64
a = _ops.empty2d(K, M, torch.float32, "cuda")
g = torch.Generator(device="cuda").manual_seed(0)
a.copy_(torch.rand(K, M, generator=g, device="cuda") + 0.5)       # all positive
q = torch.rand(K, N, generator=g, device="cuda") + 0.5
ref = a.double().T @ q.double()
e_a = _ops.h2_exponent(a)
out = _ops.gemm_h3s_t(a, e_a, _ops.split_h2(q, trans=True))
pre = _ops.gemm_h3(_ops.split_h2(a), _ops.split_h2(q, trans=True), ta=True)
tf = _ops.gemm(a, q, True, False)
rel = lambda x: ((x.double() - ref) / ref).mean().item()
print(f"chain {os.environ.get('SKP_H3_MAXCHAIN')} chunk {os.environ.get('SKP_H3_CHUNK')}: mean rel "
      f"error 3xFP16-s {rel(out):+.3e}  3xFP16 pre-split {rel(pre):+.3e}  3xTF32 {rel(tf):+.3e}")
