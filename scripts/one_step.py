"""One warm-up + one timed rsvd_sharded step of a bench config (for ncu
launch lists: python scripts/one_step.py C5).  The launches of the second
step are the step's kernel list."""
import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2605_09755_b200 import distributed as D, _engine

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"])
dev = torch.device("cuda", 0)
if cfg.get("nystrom"):
    from paper_2605_09755_b200 import datagen, power
    x, h = bench.c4_points(cfg)
    kmat = datagen.rbf_kernel_gpu(x, h, device=dev)
    spec = bench.nystrom_spec(cfg)
    for i in range(2):
        torch.cuda.synchronize()
        power._check_psd_dev(kmat)
        D.nystrom_sharded(kmat, spec, 0, cfg["n"], _engine.LOCAL)
        torch.cuda.synchronize()
        print("step", i, flush=True)
    sys.exit(0)
a = bench.make_input(cfg, 0, cfg["m"], dev)
spec = bench.spec_of(cfg, seed=cfg.get("seed", 3))
for i in range(2):
    t = {}
    torch.cuda.synchronize()
    D.rsvd_sharded(a, spec, cfg["m"], _engine.LOCAL, t, with_error=False)
    torch.cuda.synchronize()
    print("step", i, {k: round(v, 2) for k, v in t.items()}, flush=True)
