import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200 import _ops
be = _ops.CudaBackend(torch.device("cuda", 0), torch.float32)
bt = _ops.empty2d(16384, 520, torch.float32, "cuda"); bt.normal_()
for f, name in ((lambda: be.gram64_rows_t(bt), "gram_f32_f64"),
                (lambda: _ops.gemm(_ops.cast(bt, torch.float64), _ops.cast(bt, torch.float64), True, False), "cast+dgemm")):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 10, "ms")
