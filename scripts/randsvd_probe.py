"""Where the step's time goes (python scripts/randsvd_probe.py [C3|C5]): CUDA events around each backend call of
_engine.randsvd / _randsvd_core (one GPU, resident input)."""
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_09755_b200 import _ops, distributed as D  # noqa: E402

acc = defaultdict(float)
cnt = defaultdict(int)
on = [False]


def wrap(name):
    f = getattr(_ops.CudaBackend, name)

    def g(self, *a, **k):
        if not on[0]:
            return f(self, *a, **k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = f(self, *a, **k)
        e1.record()
        e1.synchronize()
        acc[name] += e0.elapsed_time(e1)
        cnt[name] += 1
        return r
    setattr(_ops.CudaBackend, name, g)


for nm in ("mm_at_big", "gram64_rows_t", "eig_desc64", "sqrt_eigs", "mm", "scale_cols_",
           "to_compute", "cols", "overflowed", "chol_inv64", "gram64", "orth_planes",
           "power_lazy_planes", "prepare", "gram64_planes", "gram64_q", "orth_dev_t",
           "power_gram", "power_gram_steps", "eig_orth64", "planes_to_compute", "dense"):
    if hasattr(_ops.CudaBackend, nm):
        wrap(nm)
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"])
spec = bench.spec_of(cfg, 3)
a = bench.make_input(cfg, 0, cfg["m"], torch.device("cuda", 0))
for _ in range(3):
    D.rsvd_sharded(a, spec, cfg["m"], bench._LocalComm(), None, with_error=False)
torch.cuda.synchronize()
on[0] = True
ph = {}
for _ in range(3):
    time.sleep(0.2)
    D.rsvd_sharded(a, spec, cfg["m"], bench._LocalComm(), ph, with_error=False)
for k in sorted(acc, key=lambda k: -acc[k]):
    print(f"{k:20s} {acc[k] / 3:8.3f} ms  ({cnt[k] // 3} calls/step)")
print({k: round(v / 3, 2) for k, v in ph.items()})
