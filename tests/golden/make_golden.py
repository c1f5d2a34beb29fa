"""Generate golden vectors from the REFERENCE package (pillarmix) for parity tests.

Run in the build container, where the read-only reference exists:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
It imports the real reference (never copied) and stores inputs + its outputs as
small .npz fixtures plus the toy detector in the reference's own .mpq format.
The GPU box has no /root/reference; tests read only these committed files.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from pillarmix import quant as Q  # noqa: E402
from pillarmix import tensor_ops as T  # noqa: E402
from pillarmix.calibration import run_calibration  # noqa: E402
from pillarmix.detector import DetectorConfig, build_toy_detector, decode_and_nms, pillarize_dataset  # noqa: E402
from pillarmix.model import PrecisionPlan, apply_plan, fold_all_bn, forward, parse_plan_label, save_model  # noqa: E402
from pillarmix.quant import DType  # noqa: E402
from pillarmix.scenes import DatasetConfig, generate_dataset  # noqa: E402

OUT = Path(__file__).resolve().parent


def quant_vectors():
    rng = np.random.default_rng(1234)
    scales = [0.03125, 0.37, 1.0, float(rng.uniform(0.01, 1.0)), 2.54 / 127.0, 1e-3, 17.0]
    data = {}
    for i, s in enumerate(scales):
        x = np.concatenate([
            rng.normal(scale=60 * s, size=4000),
            rng.uniform(-140 * s, 140 * s, size=2000),
            (rng.integers(-130, 130, size=2000) + 0.5) * s,           # exact ties (as far as f32 allows)
            (rng.integers(-130, 130, size=1000) + 0.5) * s * (1 + rng.normal(scale=1e-7, size=1000)),
            np.array([0.0, -0.0, 1e30, -1e30, 127.5 * s, -128.5 * s, 127.49 * s, -128.49 * s]),
        ]).astype(np.float32)
        qp = Q.QuantParams(scale=s)
        data[f"x{i}"] = x
        data[f"scale{i}"] = np.float64(s)
        data[f"codes{i}"] = Q.quantize(x, qp)
        data[f"fq{i}"] = Q.fake_quant(x, qp)
    f = np.concatenate([rng.normal(scale=1e3, size=5000), rng.normal(scale=1e-5, size=2000),
                        np.array([65519.0, 65520.0, 65504.0, 1e6, -1e6, 3e-8, 2049.0, 1.0, 6e-5])]).astype(np.float32)
    data["fp16_in"] = f
    data["fp16_out"] = Q.fp16_roundtrip(f)
    w = rng.normal(size=(8, 5, 3, 3)).astype(np.float32)
    w[3] *= 40.0
    w[5] = 0.0
    pc = Q.weight_quant_params(w, per_channel=True)
    data["w"] = w
    data["w_scales_pc"] = pc.scales
    data["w_fq_pc"] = Q.fake_quant_per_channel(w, pc)
    pt = Q.weight_quant_params(w)
    data["w_scale_pt"] = np.float64(pt.scale)
    data["w_fq_pt"] = Q.fake_quant(w, pt)
    mm = rng.normal(size=(1000,)).astype(np.float32)
    obs = Q.observe(Q.MinMaxObserver(), mm)
    data["obs_in"] = mm
    data["obs_minmax"] = np.array([obs.running_min, obs.running_max])
    np.savez_compressed(OUT / "ref_quant.npz", **data)


def ops_vectors():
    rng = np.random.default_rng(99)
    data = {}
    cases = [((1, 3, 9, 7), (4, 3, 3, 3), (1, 1), (1, 1)), ((2, 5, 8, 8), (6, 5, 3, 3), (2, 2), (1, 1)),
             ((1, 4, 6, 5), (3, 4, 1, 1), (1, 1), (0, 0)), ((1, 2, 7, 9), (5, 2, 3, 2), (2, 1), (0, 1))]
    for i, (xs, ws, st, pd) in enumerate(cases):
        x = rng.normal(size=xs).astype(np.float32)
        w = rng.normal(size=ws).astype(np.float32)
        b = rng.normal(size=ws[0]).astype(np.float32)
        data[f"conv{i}_x"], data[f"conv{i}_w"], data[f"conv{i}_b"] = x, w, b
        data[f"conv{i}_stride"], data[f"conv{i}_pad"] = np.array(st), np.array(pd)
        data[f"conv{i}_y"] = T.conv2d(x, w, b, T.ConvParams(stride=st, padding=pd))
    x = rng.normal(size=(7, 6)).astype(np.float32)
    w = rng.normal(size=(4, 6)).astype(np.float32)
    b = rng.normal(size=4).astype(np.float32)
    data["lin_x"], data["lin_w"], data["lin_b"], data["lin_y"] = x, w, b, T.linear(x, w, b)
    feats = rng.normal(size=(5, 4, 3)).astype(np.float32)
    mask = rng.random((5, 4)) < 0.6
    mask[:, 0] = True
    data["mop_f"], data["mop_m"], data["mop_y"] = feats, mask, T.max_over_points(feats, mask)
    cells = rng.choice(8 * 9, size=10, replace=False)
    coords = np.stack([cells // 9, cells % 9], axis=1)
    f2 = rng.normal(size=(10, 6)).astype(np.float32)
    data["sc_f"], data["sc_c"], data["sc_y"] = f2, coords, T.scatter_pillars(f2, coords, (8, 9))
    np.savez_compressed(OUT / "ref_ops.npz", **data)


def toy_vectors():
    cfg = DetectorConfig()
    graph = build_toy_detector(cfg, seed=0)
    save_model(graph, OUT / "toy")
    scenes = generate_dataset(DatasetConfig(size=6), seed=3)
    # one dense scene so that pillars overflow max_points (first-come truncation)
    rng = np.random.default_rng(5)
    dense = np.concatenate([rng.uniform(5.0, 6.0, size=(60, 2)), rng.uniform(0, 1, size=(60, 1))], axis=1)
    dense = np.concatenate([dense, scenes[0].points], axis=0).astype(np.float32)
    from pillarmix.scenes import Scene

    scenes = scenes + [Scene(points=dense, boxes=np.zeros((0, 4), np.float32), classes=np.zeros(0, np.int64),
                             difficulty=np.zeros(0, dtype=object))]
    samples = pillarize_dataset(scenes, cfg)
    data = {}
    for i, (sc, sm) in enumerate(zip(scenes, samples)):
        data[f"pts{i}"] = sc.points
        data[f"feat{i}"] = sm.features
        data[f"mask{i}"] = sm.point_mask
        data[f"coords{i}"] = sm.coords
    stats = run_calibration(graph, samples[:4], seed=0)
    stats_pc = run_calibration(graph, samples[:4], seed=0, per_channel_weights=True)
    for idx in stats.indices():
        data[f"stat{idx}_minmax"] = np.array([stats[idx].observer.running_min, stats[idx].observer.running_max])
        data[f"stat{idx}_act"] = np.float64(stats[idx].act_qp.scale)
        data[f"stat{idx}_w"] = np.float64(stats[idx].weight_qp.scale)
        data[f"statpc{idx}_w"] = stats_pc[idx].weight_qp.scales
    folded = fold_all_bn(graph)
    plans = {"FP32": PrecisionPlan(), "INT8": PrecisionPlan(default=DType.INT8),
             "FP16_1_12_3": parse_plan_label("FP16: 1,12,3"), "FP16": PrecisionPlan(default=DType.FP16)}
    for pname, plan in plans.items():
        planned = apply_plan(folded, plan)
        for i, sm in enumerate(samples):
            cls_map, reg_map = forward(planned, sm, stats=stats)
            data[f"out_{pname}_{i}_cls"] = cls_map
            data[f"out_{pname}_{i}_reg"] = reg_map
    # per-channel INT8 and unfolded-BN FP32 forwards
    for i, sm in enumerate(samples[:3]):
        c, r = forward(apply_plan(folded, PrecisionPlan(default=DType.INT8)), sm, stats=stats_pc)
        data[f"out_INT8PC_{i}_cls"], data[f"out_INT8PC_{i}_reg"] = c, r
        c, r = forward(graph, sm)
        data[f"out_UNFOLDED_{i}_cls"], data[f"out_UNFOLDED_{i}_reg"] = c, r
    # decode on the FP32 outputs, lowered thresholds so there are detections
    for i in range(len(samples)):
        cls_map = data[f"out_FP32_{i}_cls"]
        reg_map = data[f"out_FP32_{i}_reg"]
        dets = decode_and_nms(cls_map, reg_map, cfg, score_thresh=0.05, iou_thresh=0.3)
        data[f"dets{i}_box"] = np.array([d.box for d in dets]).reshape(-1, 4)
        data[f"dets{i}_cls"] = np.array([d.class_id for d in dets], np.int64)
        data[f"dets{i}_score"] = np.array([d.score for d in dets])
    np.savez_compressed(OUT / "ref_toy.npz", **data)
    (OUT / "ref_toy_meta.json").write_text(json.dumps({
        "n_samples": len(samples), "calib_samples": 4, "plans": list(plans),
        "detector": {"grid": list(cfg.grid), "field_size": cfg.field_size,
                     "max_points_per_pillar": cfg.max_points_per_pillar, "base_size": cfg.base_size},
        "decode": {"score_thresh": 0.05, "iou_thresh": 0.3}}, indent=2) + "\n")


if __name__ == "__main__":
    quant_vectors()
    ops_vectors()
    toy_vectors()
    for p in sorted(OUT.iterdir()):
        print(p.name, p.stat().st_size)
