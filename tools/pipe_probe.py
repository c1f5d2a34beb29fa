"""Timing probe for the streaming path: graph alone, H2D alone, pipelined."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402
from paper_2601_12638_b200 import distributed as D  # noqa: E402


def ev_time(fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cfg = pm.PointPillarsConfig(max_pillars=16000)
graph = pm.build_pointpillars(cfg, seed=0)
stats = pm.calibrate_frames(graph, [pm.make_frame(120000, 900 + i, cfg, 0.01) for i in range(2)], cfg)
B = 32
frames = pm.make_frames(B, 1000, cfg, (60000, 150000))
eng = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=B, max_points_per_frame=150000)
eng.load_points(frames)
eng.capture()
print("graph alone ms", ev_time(eng.run, 10))
host = torch.from_numpy(np.concatenate(frames)).pin_memory()
dst = eng.cg.points[: host.shape[0]]
print("h2d alone ms", ev_time(lambda: dst.copy_(host, non_blocking=True), 10), "bytes", host.numel() * 4)
offs = np.zeros(B + 1, np.int64)
offs[1:] = np.cumsum([len(f) for f in frames])
hoffs = torch.from_numpy(offs).pin_memory()
pipe = pm.PipelinedEngine(eng)
rec = D.pack_topk(eng.topk())
outs = [torch.empty(rec.shape, dtype=rec.dtype).pin_memory() for _ in range(2)]
for K in (5, 20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    pipe.run([(host, hoffs)] * K, [outs[i % 2] for i in range(K)], D.pack_topk)
    b.record()
    torch.cuda.synchronize()
    print("pipelined K", K, "ms/step", a.elapsed_time(b) / K)
