"""Per-rank step time at N ranks, emulated on one GPU: the rank's m/N-row slab
run through rsvd_sharded with a no-op all-reduce (the real all-reduces are
l x r2, r2 x r2 and n x r2 over NVLink: < 0.2 ms per step at C3).  Shows the
replicated (m-independent) part that bounds strong scaling."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_09755_b200 import distributed as D  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"])
spec = bench.spec_of(cfg, 3)
dev = torch.device("cuda", 0)
for N in (1, 2, 4, 8):
    row0, rows = D.shard_rows(cfg["m"], N, 0)
    a = bench.make_input(cfg, row0, rows, dev)
    for _ in range(3):
        D.rsvd_sharded(a, spec, cfg["m"], bench._LocalComm(), None, with_error=False)
    torch.cuda.synchronize()
    ph = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    time.sleep(0.3)
    e0.record()
    for _ in range(5):
        D.rsvd_sharded(a, spec, cfg["m"], bench._LocalComm(), ph, with_error=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"N={N} rows={rows}: {ms:.2f} ms/step  " +
          " ".join(f"{k}={v / 5:.2f}" for k, v in ph.items()), flush=True)
    del a
    torch.cuda.empty_cache()
