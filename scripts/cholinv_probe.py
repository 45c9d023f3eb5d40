"""Fused Cholesky + inverse: accuracy and time at the CholeskyQR sizes."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _lib, _ops
def spd(n, cond, seed):
    rng = np.random.default_rng(seed)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    return (q * np.logspace(0, -np.log10(cond), n)) @ q.T
for n in (1, 7, 32, 33, 100, 520, 544, 1050):
    g = spd(n, 1e6, n)
    t = torch.from_numpy(g).cuda()
    x = torch.empty_like(t)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    wsb = _lib.load().skp_cholinv_ws_bytes(n)
    ws = _ops.workspace(t.device, wsb)
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.call("skp_cholinv_f64", _ops.ptr(t), n, n, 1e-9, 0.0, _ops.ptr(x), _ops.ptr(info), _ops.ptr(ws), wsb, st)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    xi = x.cpu().numpy(); L = np.linalg.cholesky(g)
    err = np.abs(xi @ L - np.eye(n)).max()
    print(f"n={n}: {e0.elapsed_time(e1)/10*1e3:.0f} us  info={int(info.item())}  |X L - I|={err:.2e}  upper0={np.all(np.triu(xi,1)==0)}", flush=True)
