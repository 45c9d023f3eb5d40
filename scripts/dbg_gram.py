import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
rng = np.random.default_rng(0)
for (m, c) in ((4000, 120), (20000, 110), (4000, 30), (65536, 96)):
    y = rng.standard_normal((m, c)).astype(np.float32)
    y /= np.linalg.norm(y, axis=0)
    yd = _ops.aligned2d(torch.from_numpy(y).cuda())
    ref = y.astype(np.float64).T @ y.astype(np.float64)
    for mode in ("auto", "fp32"):
        g = _ops.gemm(yd, yd, ta=True, mode=mode).double().cpu().numpy()
        print(m, c, mode, "gram err %.2e" % np.abs(g - ref).max(), "diag err %.2e" % np.abs(np.diag(g) - np.diag(ref)).max(), flush=True)
    x = rng.standard_normal((c, c)).astype(np.float32)
    xd = _ops.aligned2d(torch.from_numpy(x).cuda())
    p = _ops.gemm(yd, xd, tb=True).double().cpu().numpy()
    pr = y.astype(np.float64) @ x.astype(np.float64).T
    print("   y x^T err %.2e (scale %.2e)" % (np.abs(p - pr).max(), np.abs(pr).max()))
