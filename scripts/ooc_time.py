"""rsvd of a host-resident C5 A forced out of core (A's row blocks streamed
from pinned host memory three times) vs the resident e2e path; sigma agree."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import power
cfg = dict(bench.CONFIGS["C5"])
dev = torch.device("cuda", 0)
a = bench.make_input(cfg, 0, cfg["m"], dev)
h = torch.empty(tuple(a.shape), dtype=torch.float32, pin_memory=True)
h.copy_(a)
del a
torch.cuda.empty_cache()
spec = bench.spec_of(cfg, cfg.get("seed", 3))
for mode in ("resident e2e", "out of core"):
    if mode == "out of core":
        power._needs_out_of_core = lambda *x: True
    skp.rsvd(h, spec)          # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = skp.rsvd(h, spec)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    s = res.sigma.numpy() if isinstance(res.sigma, torch.Tensor) else res.sigma
    print(f"{mode}: {t * 1e3:.1f} ms  sigma_1 {s[0]:.9f} sigma_k {s[cfg['k'] - 1]:.9f}", flush=True)
