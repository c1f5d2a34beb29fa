"""Batch-1 latency of the whole captured pipeline (config 3, 120k points) per plan.

    python tools/b1_latency.py                 # p50/p99 over 200 graph replays per plan
    python tools/b1_latency.py --ncu 3         # just 3 replays of the mixed plan (for an ncu launch list)
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2601_12638_b200 as pm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ncu", type=int, default=0)
    ap.add_argument("--plans", default="FP16: 2,18,19,20;INT8;FP16")
    args = ap.parse_args()
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=0)
    stats = pm.calibrate_frames(graph, [pm.make_frame(120000, 900 + i, cfg, 0.01) for i in range(2)], cfg)
    if args.ncu:
        e = pm.PointPillarsEngine(graph, args.plans.split(";")[0], stats, cfg, batch=1, max_points_per_frame=120000)
        e.load_points([pm.make_frame(120000, 77, cfg)])
        e.capture()
        for _ in range(args.ncu):
            e.run()
        torch.cuda.synchronize()
        return
    out = {}
    for label in args.plans.split(";"):
        p50, p99 = bench.b1_latency(pm, graph, stats, cfg, label, 120000, 77)
        out[label] = {"p50_ms": round(p50, 4), "p99_ms": round(p99, 4)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
