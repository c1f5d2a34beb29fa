"""Per-op device times of the batch-1 mixed pipeline (config 3, 120k points)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402

cfg = pm.PointPillarsConfig(max_pillars=16000)
graph = pm.build_pointpillars(cfg, seed=0)
stats = pm.calibrate_frames(graph, [pm.make_frame(120000, 900 + i, cfg, 0.01) for i in range(2)], cfg)
e = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=1, max_points_per_frame=120000)
e.load_points([pm.make_frame(120000, 77, cfg)])
ops = e.cg.timed_ops(reps=20)
tot = sum(ops.values())
for k, v in ops.items():
    print(f"{k:32s} {v * 1e3:8.1f} us")
print(f"{'sum':32s} {tot * 1e3:8.1f} us")
