"""3xFP16 (pre-split) vs 3xTF32 GEMMs at the C3 power-iteration shapes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops


def timeit(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


m, l, r2 = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (262144, 4000, 520)))
torch.manual_seed(0)
at = _ops.empty2d(m, l, torch.float32, "cuda"); at.normal_()
z = _ops.empty2d(l, r2, torch.float32, "cuda"); z.normal_()
y = _ops.empty2d(m, r2, torch.float32, "cuda"); y.normal_()
fl = 2.0 * m * l * r2
sa = _ops.split_h2(at)
t = timeit(lambda: _ops.split_h2(at, out=sa))
print(f"split A~ ({m}x{l}): {t:.3f} ms  {2 * m * l * 4 / t / 1e6:.0f} GB/s moved", flush=True)
sz = _ops.split_h2(z, trans=True)
t = timeit(lambda: _ops.split_h2(z, trans=True, out=sz))
print(f"split Z^T ({l}x{r2}): {t:.3f} ms", flush=True)
sy = _ops.split_h2(y, trans=True)
t = timeit(lambda: _ops.split_h2(y, trans=True, out=sy))
print(f"split Y^T ({m}x{r2}): {t:.3f} ms  {2 * m * r2 * 4 / t / 1e6:.0f} GB/s moved", flush=True)
out = _ops.empty2d(m, r2, torch.float32, "cuda")
t1 = timeit(lambda: _ops.gemm(at, z, out=out))
ref = out.clone()
t2 = timeit(lambda: _ops.gemm_h3(sa, sz, out=out))
err = ((out.double() - ref.double()).abs().max() / ref.double().abs().max()).item()
print(f"NN  A~ Z : 3xTF32 {t1:.3f} ms ({fl / t1 / 1e9:.0f} TF/s)  3xFP16 {t2:.3f} ms "
      f"({fl / t2 / 1e9:.0f} TF/s)  max rel diff {err:.2e}", flush=True)
zo = _ops.empty2d(l, r2, torch.float32, "cuda")
t1 = timeit(lambda: _ops.gemm(at, y, True, False, out=zo))
ref = zo.clone()
t2 = timeit(lambda: _ops.gemm_h3(sa, sy, ta=True, out=zo))
err = ((zo.double() - ref.double()).abs().max() / ref.double().abs().max()).item()
print(f"TN  A~^T Y: 3xTF32 {t1:.3f} ms ({fl / t1 / 1e9:.0f} TF/s)  3xFP16 {t2:.3f} ms "
      f"({fl / t2 / 1e9:.0f} TF/s)  max rel diff {err:.2e}", flush=True)
