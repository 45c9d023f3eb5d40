import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
be = _ops.CudaBackend("cuda", torch.float32)
for n, c in [(32768, 1050), (16384, 520)]:
    bt = torch.randn(n, c, device="cuda")
    be.gram64_rows_t(bt); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): g = be.gram64_rows_t(bt)
    e1.record(); torch.cuda.synchronize()
    ref = bt.double().T @ bt.double()
    print(n, c, "ms %.3f" % (e0.elapsed_time(e1) / 5), "err %.2e" % ((g - ref).abs().max() / ref.abs().max()).item())
