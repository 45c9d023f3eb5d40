"""K5 (fused Cholesky + inverse, fp64) time and accuracy at n: python scripts/cholinv_time.py 520 1050"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _lib, _ops
for n in [int(v) for v in sys.argv[1:]] or [520]:
    rng = np.random.default_rng(1)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    g = (q * np.logspace(0, -6, n)) @ q.T
    g = (g + g.T) / 2
    t = torch.from_numpy(g).cuda()
    x = torch.empty_like(t)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    wsb = _lib.load().skp_cholinv_ws_bytes(n)
    ws = _ops.workspace(t.device, wsb)
    st = torch.cuda.current_stream().cuda_stream
    run = lambda: _lib.call("skp_cholinv_f64", _ops.ptr(t), n, n, 1e-9, 0.0, _ops.ptr(x),
                            _ops.ptr(info), _ops.ptr(ws), wsb, st)
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    xi = x.cpu().numpy()
    lm = np.linalg.cholesky(g)
    print(f"n={n}: {e0.elapsed_time(e1) / 20:.3f} ms  info={int(info.item())}  "
          f"|X L - I|={np.abs(xi @ lm - np.eye(n)).max():.2e}")
