"""Debug: SYRK correctness per tile and the sketch-space power iteration's
lazy flags on a reduced C3-structured input."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops, datagen, power, _engine
import paper_2605_09755_b200 as skp

torch.cuda.set_device(0)
for (N, K) in [(300, 5000), (1000, 20000), (4000, 8192)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(K, N, generator=g, device="cuda")
    out = _ops.syrk_h3(_ops.split_h2(a))
    ref = a.double().T @ a.double()
    ab = a.double().abs()
    refabs = ab.T @ ab
    err = (out.double() - ref).abs() / refabs
    print(N, K, "max rel-to-abs err", err.max().item(), "at", np.unravel_index(err.argmax().item(), err.shape),
          "diag rel", ((torch.diagonal(out).double() - torch.diagonal(ref)) / torch.diagonal(ref)).abs().max().item())
    T = 128
    nt = (N + T - 1) // T
    bad = [(i, j, round(err[i*T:(i+1)*T, j*T:(j+1)*T].max().item(), 8)) for i in range(nt) for j in range(nt)
           if err[i*T:(i+1)*T, j*T:(j+1)*T].max().item() > 1e-4]
    print("  bad tiles:", bad[:20])

m, n, l, r2, k, q = 16384, 4096, 1000, 120, 100, 3
spec_v = np.arange(1.0, 2048 + 1.0) ** -0.5
a_dev = datagen.lowrank_plus_noise_gpu(m, n, spec_v, 1e-6, seed=3)
spec = skp.RangeFinderSpec(k=k, l=l, r1=l, r2=r2, q=q, eps=0.5, seed=3, s=8)
be = _ops.CudaBackend(a_dev.device, torch.float32)
orig = _ops.CudaBackend.chol_inv64
def traced(self, g, rel_tol, lazy=False, shift=0.0):
    x = orig(self, g, rel_tol, lazy=lazy, shift=shift)
    torch.cuda.synchronize()
    ev = torch.linalg.eigvalsh(g)
    print("  chol_inv64 n=%d lazy=%s shift=%g fail=%s  eig min %.3e max %.3e  nan=%s" % (
        g.shape[0], lazy, shift, self.fail.tolist(), ev.min().item(), ev.max().item(), bool(torch.isnan(g).any())))
    return x
_ops.CudaBackend.chol_inv64 = traced
orig_pg = _ops.CudaBackend.power_gram
def pg(self, comm, atil, omega, q, shift):
    print("power_gram: atil", atil.rows, atil.cols, atil.ld, "e", atil.e.tolist(), "omega", tuple(omega.shape))
    g = _ops.syrk_h3(atil)
    print("  G finite", bool(torch.isfinite(g).all()), "max", g.abs().max().item(), "diag min", torch.diagonal(g).min().item())
    return orig_pg(self, comm, atil, omega, q, shift)
_ops.CudaBackend.power_gram = pg
res, rel = skp.rsvd(a_dev, spec, with_error=True)
print("rel", rel)
