"""Device->host bandwidth into pinned memory: one copy, chunked over streams, reused buffer."""
import time
import torch
n = 4 << 30
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
d.fill_(1.0)


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
print(f"D2H pinned (pin_memory) single: {n / t(lambda: h.copy_(d, non_blocking=True)) / 1e9:.1f} GB/s", flush=True)
h2 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
print(f"D2H pinned (pin_memory=True alloc) single: {n / t(lambda: h2.copy_(d, non_blocking=True)) / 1e9:.1f} GB/s", flush=True)
for ns in (2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]

    def multi():
        ch = h.numel() // ns
        for i, s in enumerate(streams):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                h[i * ch:(i + 1) * ch].copy_(d[i * ch:(i + 1) * ch], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
    print(f"D2H pinned {ns} streams: {n / t(multi) / 1e9:.1f} GB/s", flush=True)
for mb in (8, 64, 512):
    ch = (mb << 20) // 4

    def chunked():
        for i in range(0, h.numel(), ch):
            h[i:i + ch].copy_(d[i:i + ch], non_blocking=True)
    print(f"D2H pinned sequential {mb} MB chunks: {n / t(chunked) / 1e9:.1f} GB/s", flush=True)
hp = torch.empty(n // 4, dtype=torch.float32)
print(f"D2H pageable: {n / t(lambda: hp.copy_(d)) / 1e9:.1f} GB/s", flush=True)
print(f"H2D pinned single: {n / t(lambda: d.copy_(h, non_blocking=True)) / 1e9:.1f} GB/s", flush=True)
