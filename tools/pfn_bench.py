"""Time the pillarize + PFN/scatter ops of the engine at the config-4 shape (batch 32)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=0)
    frames = pm.make_frames(B, 1000, cfg, (60000, 150000))
    stats = pm.calibrate_frames(graph, frames[:2], cfg)
    eng = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=B, max_points_per_frame=150000)
    eng.load_points(frames)
    for _ in range(3):
        eng.run()
    ms = eng.cg.timed_launch(reps=5)
    for k, v in ms.items():
        if not k.startswith("conv"):
            print(f"{k:30s} {v * 1e3:9.1f} us")


if __name__ == "__main__":
    main()
