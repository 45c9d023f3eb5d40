import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops, datagen
from paper_2605_09755_b200._ops import split_h2, gemm_h3, gemm_h3_emit_t, cast, symmetrize_, F64
import paper_2605_09755_b200 as skp

def planes_f32(s):
    e = int(s.e[0].item())
    return (s.hi.float() + s.lo.float())[:, :s.cols] * 2.0 ** -e

m, n, l, r2, k, q = 16384, 4096, 1000, 120, 100, 3
spec_v = np.arange(1.0, 2048 + 1.0) ** -0.5
a_dev = datagen.lowrank_plus_noise_gpu(m, n, spec_v, 1e-6, seed=3)
spec = skp.RangeFinderSpec(k=k, l=l, r1=l, r2=r2, q=q, eps=0.5, seed=3, s=8)

def pg(self, comm, atil, omega, q, shift):
    g = _ops.syrk_h3(atil)
    gs = split_h2(g)
    G = g.double()
    W = omega.double()
    wt = split_h2(omega, trans=True)
    for it in range(q):
        vt = gemm_h3_emit_t(gs, wt)
        V = planes_f32(vt).double().T
        Vref = G @ planes_f32(wt).double().T
        print(it, "wt.e", wt.e.tolist(), "vt.e", vt.e.tolist(), "gs.e", gs.e.tolist(),
              "|V| %.3e  err %.3e" % (Vref.abs().max().item(), (V - Vref).abs().max().item()))
        mg = cast(gemm_h3(wt, vt), F64)
        Mref = planes_f32(wt).double() @ V
        print("   |M| %.3e err %.3e" % (Mref.abs().max().item(), (mg - Mref).abs().max().item()))
        symmetrize_(mg)
        x = self.chol_inv64(mg, 0.0, lazy=True, shift=shift)
        xs = split_h2(self.to_compute(x))
        wt2 = gemm_h3_emit_t(vt, xs, ta=True, out=wt)
        Wn = planes_f32(wt2).double().T
        Wref = V @ x.double().T
        print("   x max %.3e xs.e %s  wt.e %s |W| %.3e err %.3e" % (x.abs().max().item(), xs.e.tolist(), wt2.e.tolist(),
              Wref.abs().max().item(), (Wn - Wref).abs().max().item()))
        wt = wt2
    return gemm_h3_emit_t(atil, wt)
_ops.CudaBackend.power_gram = pg
res, rel = skp.rsvd(a_dev, spec, with_error=True)
print("rel", rel)
