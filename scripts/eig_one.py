import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200._ops import CudaBackend
be = CudaBackend(torch.device("cuda", 0), torch.float64)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 520
rng = np.random.default_rng(n)
u, _ = np.linalg.qr(rng.standard_normal((n, n)))
g = (u * (np.arange(1, n + 1) ** -1.0)) @ u.T
t = torch.from_numpy((g + g.T) / 2).cuda()
for _ in range(2):
    be.eig_desc64(t)
torch.cuda.synchronize()
