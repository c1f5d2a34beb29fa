"""Throughput of the config-4 step with 1, 2 or 3 captured graph instances in flight on
separate streams (each instance owns its buffers; steps alternate between them)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402

cfg = pm.PointPillarsConfig(max_pillars=16000)
graph = pm.build_pointpillars(cfg, seed=0)
calib = [pm.make_frame(120000, 900 + i, cfg, outlier_frac=0.01) for i in range(2)]
stats = pm.calibrate_frames(graph, calib, cfg, per_channel_weights=True)
frames = pm.make_frames(32, 1000, cfg, (60000, 150000))
res = {}
engines = []
for n in (1, 2, 3):
    while len(engines) < n:
        e = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=32, max_points_per_frame=150000)
        e.load_points(frames)
        e.capture()
        engines.append(e)
    streams = [torch.cuda.Stream() for _ in range(n)]
    for _ in range(3):
        for e, s in zip(engines[:n], streams):
            with torch.cuda.stream(s):
                e.run()
    torch.cuda.synchronize()
    steps = 60
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in streams:
        s.wait_event(a)
    for i in range(steps):
        k = i % n
        with torch.cuda.stream(streams[k]):
            engines[k].run()
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    res[n] = {"ms_per_step": round(ms, 4), "frames_per_s": round(32 / ms * 1e3, 1)}
print(json.dumps(res))
