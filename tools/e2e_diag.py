"""Diagnostic (not a bench number): the bench's pipelined e2e loop with the full 52.7 MB
H2D per step vs the same loop copying only the offsets (the device slots already hold
the points from the warm-up, so the graphs do identical work) vs graph replays alone --
separates the copy's cost from the pipeline's structure."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402

cfg = pm.PointPillarsConfig(max_pillars=16000)
graph = pm.build_pointpillars(cfg, seed=0)
stats = pm.calibrate_frames(graph, [pm.make_frame(120000, 900 + i, cfg, 0.01) for i in range(2)], cfg)
B = 32
frames = pm.make_frames(B, 1000, cfg, (60000, 150000))
engs = []
for _ in range(2):
    e = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=B, max_points_per_frame=150000)
    e.load_points(frames)
    engs.append(e)
host_pts = torch.from_numpy(np.concatenate(frames)).pin_memory()
offs = np.zeros(B + 1, np.int64)
offs[1:] = np.cumsum([len(f) for f in frames])
host_offs = torch.from_numpy(offs).pin_memory()
pipe = pm.PipelinedEngine(engs[0], engs[1])
rec = pipe.slots[0][2]
outs = [torch.empty(rec.shape, dtype=rec.dtype).pin_memory() for _ in range(2)]
K = 50


def timed(batches):
    pipe.run(batches[:5], [outs[i % 2] for i in range(5)])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pipe.run(batches, [outs[i % 2] for i in range(len(batches))])
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / len(batches)


full = [(host_pts, host_offs)] * K
tiny = [(host_pts[:1024], host_offs)] * K
for _ in range(2):
    print(f"full H2D {timed(full):.4f} ms/step  offsets-only H2D {timed(tiny):.4f} ms/step", flush=True)
# graph replays alone, alternating engines on two streams
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
for e in engs:
    e.capture()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(K):
    with torch.cuda.stream(streams[i % 2]):
        engs[i % 2].run()
for s in streams:
    torch.cuda.current_stream().wait_stream(s)
b.record()
torch.cuda.synchronize()
print(f"graphs only {a.elapsed_time(b) / K:.4f} ms/step")
