"""K2 output digest on seeded inputs (A/B variants must print the same digest)."""
import hashlib, sys
import torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch
for (m, n, l) in ((4099, 16384, 4000), (2051, 32768, 8000), (1030, 9000, 1200)):
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(m, n, device="cuda", generator=g)
    op = make_sketch("countsketch", n, l, 11, s=8)
    got = op.right_permuted(a)
    out = got[0] if isinstance(got, tuple) else got
    torch.cuda.synchronize()
    print(m, n, l, hashlib.sha256(out.contiguous().cpu().numpy().tobytes()).hexdigest()[:16])
