"""Batch-1 whole-graph timeline of the tcgen05 conv launches (trace build only):
per launch, when its first CTA entered, when griddepcontrol.wait returned (the
previous kernel's data visible), when its CTAs exited -- relative to the first conv
CTA of one graph replay, next to the replay's event-timed duration.

    PMX_TRACE_BUILD=1 PMX_BUILD_OUT=paper_2601_12638_b200/libpmx_trace.so \\
        python -m paper_2601_12638_b200._build
    PMX_LIB=paper_2601_12638_b200/libpmx_trace.so python tools/b1_timeline.py [--plan LABEL]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402
from paper_2601_12638_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default=pm.MIXED_PLAN_LABEL)
    ap.add_argument("--points", type=int, default=120000)
    ap.add_argument("--batch", type=int, default=1)
    args = ap.parse_args()
    lib = N.load()
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=0)
    stats = pm.calibrate_frames(graph, [pm.make_frame(args.points, 900 + i, cfg, 0.01) for i in range(2)], cfg)
    eng = pm.PointPillarsEngine(graph, args.plan, stats, cfg, batch=args.batch, max_points_per_frame=args.points)
    eng.load_points([pm.make_frame(args.points, 77 + i, cfg) for i in range(args.batch)])
    buf = torch.zeros(1 + 4 * 40000, dtype=torch.int64, device="cuda")
    lib.pmx_debug_timeline(buf.data_ptr())
    eng.capture()
    lib.pmx_debug_timeline(None)
    names = [n for n, _ in eng.cg.ops]
    for _ in range(20):
        eng.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    buf.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.run()
    b.record()
    torch.cuda.synchronize()
    r = buf.cpu().numpy().view(np.uint64)
    n = int(r[0])
    rec = r[1:1 + 4 * n].reshape(n, 4).astype(np.int64)
    tags = rec[:, 0] >> 32
    t0 = rec[:, 1].min()
    print(f"graph replay {a.elapsed_time(b) * 1e3:.1f} us (p50 of 50: {np.percentile(ts, 50) * 1e3:.1f} us); "
          f"{n} conv CTAs; conv ops in graph order: {[x for x in names if x.startswith('conv')]}")
    print(f"{'tag':>4} {'ctas':>5} {'entry0':>8} {'entryN':>8} {'wait0':>8} {'waitN':>8} {'exit0':>8} {'exitN':>8}"
          f" {'run':>6} {'gap':>6}")
    prev_exit = None
    rows = []
    for t in np.unique(tags):
        m = rec[tags == t]
        rows.append((m[:, 1].min() - t0, t, m))
    for _, t, m in sorted(rows, key=lambda x: x[0]):
        e0, eN = (m[:, 1].min() - t0) / 1e3, (m[:, 1].max() - t0) / 1e3
        w0, wN = (m[:, 2].min() - t0) / 1e3, (m[:, 2].max() - t0) / 1e3
        x0, xN = (m[:, 3].min() - t0) / 1e3, (m[:, 3].max() - t0) / 1e3
        gap = w0 - prev_exit if prev_exit is not None else 0.0
        print(f"{t:4d} {len(m):5d} {e0:8.2f} {eN:8.2f} {w0:8.2f} {wN:8.2f} {x0:8.2f} {xN:8.2f} {xN - w0:6.2f} {gap:6.2f}")
        prev_exit = xN


if __name__ == "__main__":
    main()
