"""randsvd's B^T = A^T Q at C3: 3xTF32 vs 3xFP16 with the in-kernel split."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops


def timeit(f, reps=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


m, n, r2 = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (262144, 16384, 520)))
torch.manual_seed(0)
a = _ops.empty2d(m, n, torch.float32, "cuda"); a.normal_()
q = _ops.empty2d(m, r2, torch.float32, "cuda"); q.normal_()
fl = 2.0 * m * n * r2
t1 = timeit(lambda: _ops.gemm(a, q, True, False))
ref = _ops.gemm(a, q, True, False)
e_a = _ops.h2_exponent(a)
t_e = timeit(lambda: _ops.h2_exponent(a))
sq = _ops.split_h2(q, trans=True)
t_s = timeit(lambda: _ops.split_h2(q, trans=True, out=sq))
ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
out = _ops.empty2d(n, r2, torch.float32, "cuda")
t2 = timeit(lambda: _ops.gemm_h3s_t(a, e_a, sq, out=out, overflow=ovf))
err = ((out.double() - ref.double()).abs().max() / ref.double().abs().max()).item()
print(f"A^T Q {n}x{r2}x{m}: 3xTF32 {t1:.3f} ms ({fl / t1 / 1e9:.0f} TF/s); 3xFP16-s {t2:.3f} ms "
      f"({fl / t2 / 1e9:.0f} TF/s) + exact max pass {t_e:.3f} ms + Q split {t_s:.3f} ms; "
      f"max rel diff {err:.2e}; overflow {int(ovf.item())}", flush=True)
# fp64 reference on 32 columns of Q (chunked over K)
ref64 = torch.zeros(n, 32, dtype=torch.float64, device="cuda")
for k0 in range(0, m, 16384):
    ref64 += a[k0:k0 + 16384].double().T @ q[k0:k0 + 16384, :32].double()
s64 = ref64.abs().max().item()
e_tf = (ref.double()[:, :32] - ref64).abs().max().item()
e_h = (out.double()[:, :32] - ref64).abs().max().item()
print(f"vs fp64 (32 cols): 3xTF32 max err {e_tf:.3e}, 3xFP16-s max err {e_h:.3e}, max|ref| {s64:.3e}, "
      f"2e-6 max|a| max|q| sqrt(K) = {2e-6 * a.abs().max().item() * q.abs().max().item() * m ** 0.5:.3e}")
