"""Parity report for the KITTI-shaped network (SURVEY §8(d) T2 protocol).

For each plan: relative L2 per head of engine vs oracle (identical weights,
stats and pillar features), the oracle's own re-association noise floor (f32 vs
f64 accumulation, same plan), and the INT8 input-code flip rate per layer
(engine vs oracle inputs quantized with the layer's scale).  Prints JSON.
    python tools/parity_report.py [--full] [--points N]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2601_12638_b200 as pm  # noqa: E402
from oracle import pillars_oracle as O  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--points", type=int, default=None)
    ap.add_argument("--plans", default="FP32;FP16;INT8;FP16: 2,18,19,20;FP16: 1,22,3")
    args = ap.parse_args()
    cfg = pm.PointPillarsConfig(max_pillars=16000) if args.full else pm.PointPillarsConfig.small(max_pillars=1500)
    n = args.points or (120000 if args.full else 3000)
    graph = pm.build_pointpillars(cfg, seed=1)
    calib = [pm.make_frame(n, 100 + i, cfg, outlier_frac=0.01) for i in range(2)]
    ranges = O.per_sample_ranges(graph, [O.pillarize_kitti(f, cfg.grid_spec())[0] for f in calib])
    stats = pm.calibration.stats_from_ranges(graph, ranges, per_channel_weights=True)
    frame = pm.make_frame(n, 7, cfg)
    sample, _ = O.pillarize_kitti(frame, cfg.grid_spec())
    psample = pm.PillarSample(sample.features, sample.point_mask, sample.coords, sample.grid)
    plans = [p.strip() for p in args.plans.split(";") if p.strip()]
    report = {"config": "full" if args.full else "small", "points": n, "pillars": int(len(sample.coords))}
    for label in plans:
        plan = pm.parse_plan_label(label)
        planned = pm.apply_plan(pm.fold_all_bn(graph), plan)
        precs = {l.index: l.precision.value for l in planned.weight_layers}
        og = O.folded_graph(planned, precs)
        seen_o, seen_e = {}, {}
        want = O.forward(og, sample, stats=stats, observe_fn=lambda l, x: seen_o.__setitem__(l.index, x))
        with O.accumulate_in(np.float64):
            want64 = O.forward(og, sample, stats=stats)
        with O.accumulate_in("int"):
            wantint = O.forward(og, sample, stats=stats)
        got = pm.forward(planned, psample, stats=stats, observe_fn=lambda l, x: seen_e.__setitem__(l.index, x))
        flips = {}
        for l in planned.weight_layers:
            if precs[l.index] != "int8" or l.index == 1:
                continue
            s = float(stats[l.index].act_qp.scale)
            a, b = O.quantize(seen_e[l.index], s), O.quantize(seen_o[l.index], s)
            flips[l.index] = float(np.mean(a != b))
        report[label] = {
            "engine_vs_ref": {h: rel(g, w) for h, g, w in zip(pm.pointpillars.HEADS, got, want)},
            "ref_f32_vs_f64": {h: rel(w, w64) for h, w, w64 in zip(pm.pointpillars.HEADS, want, want64)},
            "engine_vs_f64": {h: rel(g, w64) for h, g, w64 in zip(pm.pointpillars.HEADS, got, want64)},
            "ref_f32_vs_int": {h: rel(w, wi) for h, w, wi in zip(pm.pointpillars.HEADS, want, wantint)},
            "engine_vs_int": {h: rel(g, wi) for h, g, wi in zip(pm.pointpillars.HEADS, got, wantint)},
            "int8_input_flip_rate": flips,
        }
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
