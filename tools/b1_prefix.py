"""In-graph cost of every op of the batch-1 step: capture the first k ops of the engine
(no side-stream branches) as one CUDA graph, replay it, and report the increment of
the p50 replay time per added op.

    PMX_NECK_STREAM=0 python tools/b1_prefix.py [--plan LABEL]
"""
import argparse
import gc
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402
from paper_2601_12638_b200 import _native as N  # noqa: E402


def p50_graph(ops, stream, reps=100):
    with torch.cuda.stream(stream):
        for _, fn in ops:
            fn(N.stream_ptr(stream))
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _, fn in ops:
                fn(N.stream_ptr(stream))
    finally:
        gc.enable()
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.percentile(ts, 50))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default=pm.MIXED_PLAN_LABEL)
    ap.add_argument("--points", type=int, default=120000)
    args = ap.parse_args()
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=0)
    stats = pm.calibrate_frames(graph, [pm.make_frame(args.points, 900 + i, cfg, 0.01) for i in range(2)], cfg)
    eng = pm.PointPillarsEngine(graph, args.plan, stats, cfg, batch=1, max_points_per_frame=args.points)
    eng.load_points([pm.make_frame(args.points, 77, cfg)])
    ops = eng.cg.ops
    stream = torch.cuda.Stream()
    prev = 0.0
    print(f"{'k':>3} {'op':40s} {'prefix us':>10} {'+us':>7}")
    for k in range(1, len(ops) + 1):
        t = p50_graph(ops[:k], stream)
        print(f"{k:3d} {ops[k - 1][0]:40s} {t:10.1f} {t - prev:7.1f}")
        prev = t


if __name__ == "__main__":
    main()
