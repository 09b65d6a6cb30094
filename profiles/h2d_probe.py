"""Host->device copy bandwidth on this box (pinned source, 8 MiB per step,
the size of C2's per-batch features): one stream vs N concurrent streams,
timed with CUDA events over 200 back-to-back copies, plus the same copy
replayed from a CUDA graph (as bench.py's e2e path issues it).  e2e at C2
moves 8.4 MB of features per 512-request batch, so this bounds bench.py's
e2e number."""
import torch

n = 8 << 20
reps = 200
src = torch.empty(n // 4).pin_memory()
dst = torch.empty(n // 4, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n // 4) // ns

    def issue():
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk],
                                                     non_blocking=True)

    for _ in range(5):
        issue()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for _ in range(reps):
        issue()
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    print(f"H2D {ns} stream(s): {reps * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")

g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    dst.copy_(src, non_blocking=True)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"H2D graph replay: {reps * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
