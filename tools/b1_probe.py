"""Batch-1 p50 of the mixed (config 3) and all-INT8 (config 2) plans, one JSON line."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2601_12638_b200 as pm  # noqa: E402

cfg = pm.PointPillarsConfig(max_pillars=16000)
graph = pm.build_pointpillars(cfg, seed=0)
calib = [pm.make_frame(120000, 900 + i, cfg, outlier_frac=0.01) for i in range(2)]
stats = pm.calibrate_frames(graph, calib, cfg, per_channel_weights=True)
out = {}
for label in ("FP16: 2,18,19,20", "INT8"):
    p50, p99 = bench.b1_latency(pm, graph, stats, cfg, pm.parse_plan_label(label), 120000, 77)
    out[label] = round(p50, 4)
print(json.dumps(out))
