"""Per-layer B200 latency table (the analogue of the paper's Table II):
each engine op of a batch-1, 120k-point frame captured in its own CUDA graph and
replayed, for the all-FP32, all-FP16 and all-INT8 plans.

    python tools/layer_latency.py [--points 120000] [--reps 200] > profiles/r1_layer_latency.md
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402
from paper_2601_12638_b200 import _native as N  # noqa: E402


def op_times(eng, reps):
    cg = eng.cg
    out = {}
    s = torch.cuda.Stream()
    for name, fn in cg.ops:
        with torch.cuda.stream(s):
            fn(N.stream_ptr(s))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(N.stream_ptr(s))
        for _ in range(10):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        out[name] = 1e3 * a.elapsed_time(b) / reps
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=120000)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--json", action="store_true")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--plans", default="FP32;FP16;INT8")
    args = ap.parse_args()
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=0)
    frames = [pm.make_frame(args.points, 5 + i, cfg) for i in range(args.batch)]
    stats = pm.calibrate_frames(graph, [pm.make_frame(args.points, 900 + i, cfg, 0.01) for i in range(2)], cfg)
    names = {l.name: l.index for l in graph.weight_layers}
    table = {}
    fused_plans = set()
    plans = args.plans.split(";")
    for label in plans:
        eng = pm.PointPillarsEngine(graph, label, stats if label != "FP32" and label != "FP16" else None, cfg,
                                    batch=args.batch, max_points_per_frame=args.points)
        eng.load_points(frames)
        eng.run()
        t = op_times(eng, args.reps)
        # small batches run the deconvs with the heads fused (ops "conv <deblock>+heads"):
        # report each under its deconv row and the heads row as included there
        if any(k.endswith("+heads") for k in t):
            t = {(k[:-len("+heads")] if k.endswith("+heads") else k): v for k, v in t.items()}
            t["conv heads(fused)"] = 0.0
            fused_plans.add(label)
        table[label] = t
    rows = []
    for op in table[plans[0]]:
        if op.startswith("conv "):
            lname = op[5:]
            idx = names.get(lname, "21-23" if "heads" in lname else "")
        elif op == "pfn":
            lname, idx = "voxel_encoder.pfn_layers.0.linear (+maxpool+scatter)", 1
        else:
            lname, idx = op, ""
        rows.append((idx, lname, *(table[p].get(op, float("nan")) for p in plans)))
    if args.json:
        print(json.dumps({"points": args.points, "rows": rows}))
        return
    print(f"B200 per-op latency, batch {args.batch}, {args.points} points/frame, 16000 pillars "
          "(us, CUDA-graph replay of one op)\n")
    print("| index | layer | " + " | ".join(plans) + " |")
    print("|---|---|" + "---|" * len(plans))
    tot = [0.0] * len(plans)
    for r in rows:
        cells = [("in 18-20" if (p in fused_plans and "heads" in str(r[1]) and r[0] == "21-23") else f"{v:.1f}")
                 for p, v in zip(plans, r[2:])]
        print(f"| {r[0]} | {r[1]} | " + " | ".join(cells) + " |")
        for i in range(len(plans)):
            tot[i] += r[2 + i]
    print("| | **sum** | " + " | ".join(f"**{t:.1f}**" for t in tot) + " |")
    if fused_plans:
        print(f"\n{', '.join(sorted(fused_plans))}: deconvs 18-20 run fused with the 1x1 heads at this batch "
              "(`pmx_deconv_heads`, the engine's choice at batch <= 2); each deconv row includes its head slice.")


if __name__ == "__main__":
    main()
