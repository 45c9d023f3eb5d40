import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _lib, _ops
n = int(sys.argv[1]) if len(sys.argv) > 1 else 520
rng = np.random.default_rng(1)
q = np.linalg.qr(rng.standard_normal((n, n)))[0]
g = (q * np.logspace(0, -6, n)) @ q.T
t = torch.from_numpy(g).cuda(); x = torch.empty_like(t)
info = torch.zeros(1, dtype=torch.int32, device="cuda")
wsb = _lib.load().skp_cholinv_ws_bytes(n); ws = _ops.workspace(t.device, wsb)
for _ in range(3):
    _lib.call("skp_cholinv_f64", _ops.ptr(t), n, n, 1e-9, 0.0, _ops.ptr(x), _ops.ptr(info), _ops.ptr(ws), wsb, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize(); print("ok", int(info.item()))
