"""H2D / D2H copy rate of 1 GiB pinned <-> device: one copy vs the same bytes split over 2 / 4 streams."""
import time

import torch

n = 1 << 27  # 1 GiB of int64
h = torch.empty(n, dtype=torch.int64).pin_memory()
h.fill_(1)
d = torch.empty(n, dtype=torch.int64, device="cuda")
for rep in range(2):
    for parts in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(parts)]
        for direction in ("h2d", "d2h"):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step = n // parts
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    a, b = i * step, (i + 1) * step
                    if direction == "h2d":
                        d[a:b].copy_(h[a:b], non_blocking=True)
                    else:
                        h[a:b].copy_(d[a:b], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"{direction} parts={parts}: {n * 8 / dt / 1e9:.1f} GB/s")
# both directions at once (full duplex)
h2 = torch.empty(n, dtype=torch.int64).pin_memory()
d2 = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"duplex: {2 * n * 8 / dt / 1e9:.1f} GB/s total")
