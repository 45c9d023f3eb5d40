import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops, datagen, power, _engine
from paper_2605_09755_b200.sketching import make_sketch, substream
import paper_2605_09755_b200 as skp
from oracle import skp_oracle as o
n, l, r2, q = 4096, 512, 64, 2
x = datagen.rbf_points(n, 16, seed=4)
h = datagen.rbf_bandwidth(x, 4096, seed=4)
kdev = datagen.rbf_kernel_gpu(x, h)
sk = make_sketch("countsketch", n, l, substream(4, 0), s=8, device="cuda")
S = torch.zeros(n, l, dtype=torch.float64, device="cuda")
S.scatter_add_(1, sk.d_cols.long(), sk.d_signs.double() / np.sqrt(8))
ct_ref = kdev.double() @ S
nf = torch.zeros(1, dtype=torch.int64, device="cuda")
got = sk.right_permuted(kdev, nonfinite=nf)
ct, perm = got
pl = perm.long()
print("C~ perm err", ((ct.double() - ct_ref[:, pl]).abs().max() / ct_ref.abs().max()).item())
ct64 = _ops.cast(ct, torch.float64)
print("cast shape", ct64.shape, ct64.stride())
wt = sk.left_t(ct64)
wt_ref = S.T @ ct_ref
print("W~' err", ((wt - wt_ref[:, pl]).abs().max() / wt_ref.abs().max()).item())
wtp = _ops.permute_rows(wt, perm)
print("W~P err", ((wtp - wt_ref[pl][:, pl]).abs().max() / wt_ref.abs().max()).item())
spec = skp.RangeFinderSpec(k=64, l=l, r1=l, r2=r2, q=q, eps=0.5, seed=4, s=8)
res = skp.nystrom_psd(kdev, spec)
kh = kdev.cpu().numpy()
print("ours", o.nystrom_rel_error(kh, res.C.cpu().numpy(), res.W.cpu().numpy()))
ospec = o.Spec(k=64, l=l, r1=l, r2=r2, q=q, seed=4, s=8)
co, wo = o.nystrom_core(kh, ospec, stabilized=False)
print("oracle literal", o.nystrom_rel_error(kh, co, wo))
om = torch.from_numpy(o.draw_omega(l, r2, o.substream(4, 1))).cuda()
wsym = (wt_ref + wt_ref.T) / 2
y = wsym @ (wsym @ om)
c = ct_ref @ y
w = y.T @ wsym @ y
print("torch literal", o.nystrom_rel_error(kh, c.cpu().numpy(), ((w + w.T) / 2).cpu().numpy()))
print("C diff vs torch", (res.C - c).abs().max().item() / c.abs().max().item())
