"""Host->device bandwidth on this box: pinned single copy, chunked multi-stream, pageable."""
import time, torch
n = 4 << 30
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
s1 = t(lambda: d.copy_(h, non_blocking=True))
print(f"pinned single copy: {n / s1 / 1e9:.1f} GB/s", flush=True)
streams = [torch.cuda.Stream() for _ in range(4)]
def multi():
    ch = h.numel() // 4
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
s2 = t(multi)
print(f"pinned 4 streams: {n / s2 / 1e9:.1f} GB/s", flush=True)
dh = torch.empty_like(h)
s3 = t(lambda: dh.copy_(d, non_blocking=True))
print(f"pinned D2H: {n / s3 / 1e9:.1f} GB/s", flush=True)
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
