"""Device Omega vs numpy: mismatch counts and timing."""
import math, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
from paper_2605_09755_b200.sketching import _host_rng, pcg64_state
for (rows, cols, seed) in [(4000, 520, 1), (2000, 110, 2), (8000, 1050, 3), (4096, 266, 4), (13, 7, 5), (40000, 520, 6)]:
    st, inc = pcg64_state(seed)
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    d64 = _ops.gaussian(st, inc, rows, cols, math.sqrt(cols), torch.float64, "cuda", fail)
    d32 = _ops.gaussian(st, inc, rows, cols, math.sqrt(cols), torch.float32, "cuda", fail)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ref = _host_rng(seed).standard_normal((rows, cols)) / math.sqrt(cols)
    th = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        _ops.gaussian(st, inc, rows, cols, math.sqrt(cols), torch.float32, "cuda", fail)
    e1.record(); torch.cuda.synchronize()
    td = e0.elapsed_time(e1) / 5
    g64 = d64.cpu().numpy(); g32 = d32.cpu().numpy()
    mm64 = np.count_nonzero(g64 != ref); mm32 = np.count_nonzero(g32 != ref.astype(np.float32))
    first = np.argwhere(g64 != ref)[:3].tolist()
    print(f"{rows}x{cols} seed {seed}: fail={int(fail.item())} mismatches f64 {mm64} f32 {mm32} first {first} "
          f"maxrel {np.max(np.abs(g64 - ref) / (np.abs(ref) + 1e-300)):.2e}  device {td:.3f} ms host {th*1e3:.1f} ms", flush=True)
