"""Where the end-to-end rsvd time goes for a host (pinned) input at C3 size."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import _convert, power
m, n = 262144, 16384
a_dev = torch.randn(m, n, device="cuda")
host = a_dev.cpu().pin_memory()
del a_dev
torch.cuda.empty_cache()
spec = skp.RangeFinderSpec(k=500, l=4000, r1=4000, r2=520, q=3, eps=0.5, s=8, seed=3)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    op = _convert.upload(host, "a", check_finite=False)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    fro2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    qb = power._range_finder_dev(op.t, spec, fro2=fro2)
    u, s, v = power._randsvd_dev(op.t, qb, check=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    U = _convert.download(u, "cpu"); S = _convert.download(s, "cpu"); V = _convert.download(v, "cpu")
    t3 = time.perf_counter()
    del op, qb, u, s, v
    print(f"upload {1e3*(t1-t0):.1f} ms ({host.numel()*4/(t1-t0)/1e9:.1f} GB/s)  compute {1e3*(t2-t1):.1f}  download {1e3*(t3-t2):.1f}", flush=True)
