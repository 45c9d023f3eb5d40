"""Accuracy of randsvd's B^T = A^T Q at C3 (K = m = 262144): sigma from the
3xTF32 / 3xFP16-s products vs an fp64 product, same Q."""
import os
import sys
import torch
sys.path.insert(0, ".")
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import _ops, datagen, power

m, n = 262144, 16384
a = datagen.c3_matrix_gpu(3, m, n, device="cuda")
spec = skp.RangeFinderSpec(k=500, l=4000, r1=4000, r2=520, q=3, eps=0.5, s=8, seed=3)
q = power._range_finder_dev(a, spec)
torch.cuda.synchronize()
bt64 = torch.zeros(n, q.shape[1], dtype=torch.float64, device="cuda")
for k0 in range(0, m, 8192):
    bt64 += a[k0:k0 + 8192].double().T @ q[k0:k0 + 8192].double()
s64 = torch.linalg.svdvals(bt64)
be = _ops.CudaBackend("cuda", torch.float32)
for name, f in [("3xTF32", lambda: _ops.gemm(a, q, True, False)),
                ("3xFP16-s", lambda: be.mm_at_big(a, q))]:
    bt = f()
    s = torch.linalg.svdvals(bt.double())
    rel = ((s - s64).abs() / s64[0]).max().item()
    d = (bt.double() - bt64).abs().max().item() / bt64.abs().max().item()
    print(f"{name}: sigma_1 {s[0].item():.9f} vs fp64 {s64[0].item():.9f}; max |dsigma|/sigma_1 "
          f"{rel:.3e}; sigma_1 rel {(s[0] - s64[0]).item() / s64[0].item():.3e}; max|dB|/max|B| {d:.3e}",
          flush=True)
qq = torch.zeros(q.shape[1], q.shape[1], dtype=torch.float64, device="cuda")
for k0 in range(0, m, 8192):
    qd = q[k0:k0 + 8192].double()
    qq += qd.T @ qd
eye = torch.eye(q.shape[1], dtype=torch.float64, device="cuda")
dq = qq - eye
print(f"final Q: max|Q^T Q - I| {dq.abs().max().item():.3e}; mean diag dev {torch.diagonal(dq).mean().item():+.3e}",
      flush=True)
