"""Raw pinned-host -> device copy bandwidth (the e2e path's ceiling), one and two streams."""
import time

import torch

n = 157_286_400  # one H frame (bytes)
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
dst2 = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"1 stream: {n / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h = n // 2
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        dst[:h].copy_(src[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        dst[h:].copy_(src[h:], non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"2 streams: {n / dt / 1e9:.1f} GB/s")
