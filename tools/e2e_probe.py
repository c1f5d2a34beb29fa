"""Repeat the bench's end-to-end pipelined measurement several times in one process."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402
from paper_2601_12638_b200 import distributed as D  # noqa: E402

cfg = pm.PointPillarsConfig(max_pillars=16000)
graph = pm.build_pointpillars(cfg, seed=0)
plan = pm.parse_plan_label(pm.MIXED_PLAN_LABEL)
stats = pm.calibrate_frames(graph, [pm.make_frame(120000, 900 + i, cfg, 0.01) for i in range(2)], cfg,
                            per_channel_weights=True)
B = 32
frames = pm.make_frames(B, 1000, cfg, (60000, 150000))
eng = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=B, max_points_per_frame=150000)
eng.load_points(frames)
eng.capture()
host_pts = torch.from_numpy(np.concatenate(frames)).pin_memory()
offs = np.zeros(B + 1, np.int64)
offs[1:] = np.cumsum([len(f) for f in frames])
host_offs = torch.from_numpy(offs).pin_memory()
rec = D.pack_topk(eng.topk())
pipe = pm.PipelinedEngine(eng)
host_recs = [torch.empty(rec.shape, dtype=rec.dtype).pin_memory() for _ in range(2)]
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(8):
    pipe.run([(host_pts, host_offs)] * 5, [host_recs[i % 2] for i in range(5)], D.pack_topk)
    torch.cuda.synchronize()
    a.record()
    pipe.run([(host_pts, host_offs)] * K, [host_recs[i % 2] for i in range(K)], D.pack_topk)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    g0 = torch.cuda.Event(enable_timing=True); g1 = torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(K):
        eng.run()
    g1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: e2e {ms:.3f} ms/step = {B / ms * 1e3:.0f} frames/s; graph only {g0.elapsed_time(g1) / K:.3f} ms")
