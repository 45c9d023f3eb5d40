"""K6 time at n (default 520) with CUDA events, and its accuracy vs numpy eigh."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200._ops import CudaBackend
be = CudaBackend(torch.device("cuda", 0), torch.float64)
for n in [int(x) for x in sys.argv[1:]] or [520]:
    rng = np.random.default_rng(n)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    g = (u * (np.arange(1, n + 1) ** -1.0)) @ u.T
    g = (g + g.T) / 2
    t = torch.from_numpy(g).cuda()
    for _ in range(3):
        w, v = be.eig_desc64(t)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        w, v = be.eig_desc64(t)
    e1.record()
    torch.cuda.synchronize()
    wr = np.sort(np.linalg.eigvalsh(g))[::-1]
    wn, vn = w.cpu().numpy(), v.cpu().numpy()
    res = np.abs(g @ vn - vn * wn).max()
    print(f"n={n}: {e0.elapsed_time(e1) / 10:.3f} ms  max|w-w_ref|={np.abs(wn - wr).max():.2e}  "
          f"max|G V - V W|={res:.2e}  |V^T V - I|={np.abs(vn.T @ vn - np.eye(n)).max():.2e}")
