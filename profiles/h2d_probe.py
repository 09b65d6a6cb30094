"""Host->device copy bandwidth on this box: one stream vs N concurrent
streams (8 MiB total per step, pinned source).  e2e at C2 moves 8.4 MB of
features per 512-request batch, so this bounds bench.py's e2e number."""
import time

import torch

n = 8 << 20
src = torch.empty(n // 4).pin_memory()
dst = torch.empty(n // 4, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n // 4) // ns
    for _ in range(3):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 50
    for _ in range(reps):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D {ns} stream(s): {reps * n / dt / 1e9:.1f} GB/s")
