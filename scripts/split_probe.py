import sys, time, torch
sys.path.insert(0, ".")
import bench
from paper_2605_09755_b200 import distributed as D
cfg = dict(bench.CONFIGS["C3"]); spec = bench.spec_of(cfg, 3); dev = torch.device("cuda", 0)
for N in [int(x) for x in sys.argv[1:]]:
    row0, rows = D.shard_rows(cfg["m"], N, 0)
    a = bench.make_input(cfg, row0, rows, dev)
    for it in range(8):
        ph = {}
        D.rsvd_sharded(a, spec, cfg["m"], bench._LocalComm(), ph, with_error=False)
        torch.cuda.synchronize()
        print(N, it, {k: round(v, 2) for k, v in ph.items()}, torch.cuda.memory_reserved() >> 20, flush=True)
    del a; torch.cuda.empty_cache()
