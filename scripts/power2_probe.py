"""Power-iteration products with 2 vs 3 fp16 products (SKP_H3_POWER2): sigma and
the projection error of the C3 rSVD, and the time of one product."""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for env in ({"SKP_H3_POWER2": "1"}, {}):
        e = dict(os.environ, **env)
        print(env, subprocess.run([sys.executable, __file__, "x"], env=e, capture_output=True,
                                  text=True).stdout.strip(), flush=True)
    sys.exit(0)
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_09755_b200 as skp
from paper_2605_09755_b200 import datagen, distributed as D
m, n = 262144, 16384
a = datagen.c3_matrix_gpu(3, m, n, device="cuda")
spec = skp.RangeFinderSpec(k=500, l=4000, r1=4000, r2=520, q=3, eps=0.5, s=8, seed=3)
class L:
    rank, world = 0, 1
    def allreduce_(self, t): return t
u, s, v, rel = D.rsvd_sharded(a, spec, m, L(), None, with_error=True)
np.save(f"/tmp/sig_{os.environ.get('SKP_H3_POWER2', '0')}.npy", s.double().cpu().numpy())
ph = {}
for _ in range(3):
    D.rsvd_sharded(a, spec, m, L(), ph, with_error=False)
print(f"rel_err {rel:.9f} sigma_1 {s[0].item():.9f} sigma_500 {s[499].item():.9f} "
      f"power {ph['power'] / 3:.2f} ms step {sum(ph.values()) / 3:.2f} ms")
if not os.environ.get("SKP_H3_POWER2"):
    s2 = np.load("/tmp/sig_1.npy")
    s3 = s.double().cpu().numpy()
    print(f"max |sigma(2 products) - sigma(3)| / sigma_1 = {np.abs(s2 - s3).max() / s3[0]:.3e}; "
          f"per-sigma relative, top 500: {(np.abs(s2[:500] - s3[:500]) / s3[:500]).max():.3e}")
