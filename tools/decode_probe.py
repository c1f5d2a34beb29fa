"""How many candidates reach the decode's final sort (the keys in the k-th key's
2048-bin histogram bin and above), per frame, for the bench's batch-1 / batch-32 frames.

    python tools/decode_probe.py [--batch 1]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--points", type=int, default=120000)
    args = ap.parse_args()
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=0)
    stats = pm.calibrate_frames(graph, [pm.make_frame(args.points, 900 + i, cfg, 0.01) for i in range(2)], cfg)
    eng = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=args.batch,
                                max_points_per_frame=args.points)
    eng.load_points([pm.make_frame(args.points, 77 + i, cfg) for i in range(args.batch)])
    eng.run()
    torch.cuda.synchronize()
    B, H, W, _ = eng.cg.heads_cat.shape
    ncand = H * W * 2
    al = lambda x: (x + 255) & ~255  # noqa: E731
    off = al(8 * B * ncand) * 2 + al(4 * B * 2048)
    cnt = eng.cg.decode_ws[off:off + 4 * B].view(torch.int32).cpu().numpy()
    print(f"batch {B}: {ncand} anchors/frame, k={cfg.topk if hasattr(cfg, 'topk') else '?'}; candidates per frame:",
          cnt.tolist()[:8], "max", int(cnt.max()))


if __name__ == "__main__":
    main()
