import os, sys, time, subprocess
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200._ops import CudaBackend
be = CudaBackend(torch.device("cuda", 0), torch.float64)
for n in (520, 1050):
    rng = np.random.default_rng(n)
    # Gram of a polynomially decaying matrix (like B B^T at C3)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = (np.arange(1, n + 1) ** -1.0)
    g = (u * lam) @ u.T
    g = (g + g.T) / 2
    t = torch.from_numpy(g).cuda()
    be.eig_desc64(t); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); w, v = be.eig_desc64(t); e1.record(); torch.cuda.synchronize()
    sw = int(be.info[1].item())
    err = np.abs(np.sort(w.cpu().numpy())[::-1] - np.sort(np.linalg.eigvalsh(g))[::-1]).max() / lam[0]
    V = v.cpu().numpy(); W = w.cpu().numpy()
    res = np.abs(g @ V - V * W).max() / lam[0]; orth = np.abs(V.T @ V - np.eye(n)).max()
    print(f"n={n} time={e0.elapsed_time(e1):.2f} ms sweeps={sw} eigerr={err:.1e} resid={res:.1e} orth={orth:.1e}", flush=True)
'''
for variant in ("tri",):
    env = dict(os.environ, SKP_SYEVJ=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print(variant, r.stdout, r.stderr[-400:], flush=True)
