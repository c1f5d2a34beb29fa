"""H2D bandwidth with the step's 52.7 MB split over 1/2/4 streams (copy engines)."""
import torch

n = 52_699_000 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    step = (n + ns - 1) // ns
    def go():
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        go()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"{ns} streams: {ms:.3f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
