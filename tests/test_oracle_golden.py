"""Pin the CPU oracle against the reference's own outputs (golden vectors made by
tests/golden/make_golden.py from the real pillarmix package).  CPU only."""

import json

import numpy as np
import pytest

from oracle import pillars_oracle as O
from tests.conftest import GOLDEN


def test_quant_codes_and_fake_quant_bit_exact(golden):
    g = golden("ref_quant.npz")
    i = 0
    while f"x{i}" in g:
        s = float(g[f"scale{i}"])
        np.testing.assert_array_equal(O.quantize(g[f"x{i}"], s), g[f"codes{i}"])
        np.testing.assert_array_equal(O.fake_quant(g[f"x{i}"], s), g[f"fq{i}"])
        i += 1
    assert i >= 5


def test_fp16_and_weight_quant(golden):
    g = golden("ref_quant.npz")
    np.testing.assert_array_equal(O.fp16_roundtrip(g["fp16_in"]), g["fp16_out"])
    pc = O.weight_scales(g["w"], per_channel=True)
    np.testing.assert_array_equal(pc, g["w_scales_pc"])
    np.testing.assert_array_equal(O.fake_quant_per_channel(g["w"], pc), g["w_fq_pc"])
    pt = O.weight_scales(g["w"], per_channel=False)
    assert pt == float(g["w_scale_pt"])
    np.testing.assert_array_equal(O.fake_quant(g["w"], pt), g["w_fq_pt"])
    lo, hi = O.minmax(g["obs_in"])
    assert (lo, hi) == tuple(g["obs_minmax"])


def test_tensor_ops(golden):
    g = golden("ref_ops.npz")
    for i in range(4):
        y = O.conv2d(g[f"conv{i}_x"], g[f"conv{i}_w"], g[f"conv{i}_b"], tuple(g[f"conv{i}_stride"]),
                     tuple(g[f"conv{i}_pad"]))
        np.testing.assert_array_equal(y, g[f"conv{i}_y"])
    np.testing.assert_array_equal(O.linear(g["lin_x"], g["lin_w"], g["lin_b"]), g["lin_y"])
    np.testing.assert_array_equal(O.max_over_points(g["mop_f"], g["mop_m"]), g["mop_y"])
    np.testing.assert_array_equal(O.scatter_pillars(g["sc_f"], g["sc_c"], (8, 9)), g["sc_y"])


def _toy():
    from paper_2601_12638_b200.model import load_model

    return load_model(GOLDEN / "toy")


def toy_stats(g, graph, per_channel=False):
    layers = {}
    for l in graph.weight_layers:
        i = l.index
        wqp = O._PCQP(g[f"statpc{i}_w"]) if per_channel else O._QP(float(g[f"stat{i}_w"]))
        mm = g[f"stat{i}_minmax"]
        layers[i] = O.LayerStats(index=i, name=l.name, observer=O._Obs(float(mm[0]), float(mm[1]), 4),
                                 act_qp=O._QP(float(g[f"stat{i}_act"])), weight_qp=wqp)
    return O.Stats(layers=layers, n_samples=4)


def test_pillarize_ref5_bit_exact(golden):
    g = golden("ref_toy.npz")
    meta = json.loads((GOLDEN / "ref_toy_meta.json").read_text())["detector"]
    for i in range(json.loads((GOLDEN / "ref_toy_meta.json").read_text())["n_samples"]):
        s = O.pillarize_ref5(g[f"pts{i}"], tuple(meta["grid"]), meta["max_points_per_pillar"], meta["field_size"])
        np.testing.assert_array_equal(s.coords, g[f"coords{i}"])
        np.testing.assert_array_equal(s.point_mask, g[f"mask{i}"])
        np.testing.assert_array_equal(s.features, g[f"feat{i}"])


PLANS = {"FP32": {}, "INT8": "int8", "FP16": "fp16", "FP16_1_12_3": {1: "fp16", 12: "fp16", 3: "fp16"}}


def _precisions(graph, plan):
    if isinstance(plan, str):
        return {l.index: plan for l in graph.weight_layers}
    if not plan:
        return {}
    return {l.index: plan.get(l.index, "int8") for l in graph.weight_layers}


@pytest.mark.parametrize("pname", list(PLANS))
def test_toy_forward_bit_exact(golden, pname):
    g = golden("ref_toy.npz")
    graph = _toy()
    stats = toy_stats(g, graph)
    n = json.loads((GOLDEN / "ref_toy_meta.json").read_text())["n_samples"]
    for i in range(n):
        sample = O.Sample(g[f"feat{i}"], g[f"mask{i}"], g[f"coords{i}"], (16, 16))
        cls_map, reg_map = O.planned_forward(graph, sample, stats, _precisions(graph, PLANS[pname]))
        np.testing.assert_array_equal(cls_map, g[f"out_{pname}_{i}_cls"])
        np.testing.assert_array_equal(reg_map, g[f"out_{pname}_{i}_reg"])


def test_toy_forward_per_channel_and_unfolded(golden):
    g = golden("ref_toy.npz")
    graph = _toy()
    stats = toy_stats(g, graph, per_channel=True)
    for i in range(3):
        sample = O.Sample(g[f"feat{i}"], g[f"mask{i}"], g[f"coords{i}"], (16, 16))
        c, r = O.planned_forward(graph, sample, stats, _precisions(graph, "int8"))
        np.testing.assert_array_equal(c, g[f"out_INT8PC_{i}_cls"])
        np.testing.assert_array_equal(r, g[f"out_INT8PC_{i}_reg"])
        c, r = O.forward(graph, sample)
        np.testing.assert_array_equal(c, g[f"out_UNFOLDED_{i}_cls"])
        np.testing.assert_array_equal(r, g[f"out_UNFOLDED_{i}_reg"])


def test_calibration_matches_reference(golden):
    g = golden("ref_toy.npz")
    graph = _toy()
    samples = [O.Sample(g[f"feat{i}"], g[f"mask{i}"], g[f"coords{i}"], (16, 16)) for i in range(4)]
    st = O.run_calibration(graph, samples)
    st_pc = O.run_calibration(graph, samples, per_channel_weights=True)
    for l in graph.weight_layers:
        i = l.index
        assert (st[i].observer.running_min, st[i].observer.running_max) == tuple(g[f"stat{i}_minmax"])
        assert st[i].act_qp.scale == float(g[f"stat{i}_act"])
        assert st[i].weight_qp.scale == float(g[f"stat{i}_w"])
        np.testing.assert_array_equal(st_pc[i].weight_qp.scales, g[f"statpc{i}_w"])


def test_toy_decode_and_nms(golden):
    g = golden("ref_toy.npz")
    meta = json.loads((GOLDEN / "ref_toy_meta.json").read_text())
    det, dec = meta["detector"], meta["decode"]
    for i in range(meta["n_samples"]):
        dets = O.decode_and_nms(g[f"out_FP32_{i}_cls"], g[f"out_FP32_{i}_reg"], det["field_size"], det["base_size"],
                                dec["score_thresh"], dec["iou_thresh"])
        boxes = np.array([d[0] for d in dets]).reshape(-1, 4)
        np.testing.assert_array_equal(boxes, g[f"dets{i}_box"])
        np.testing.assert_array_equal(np.array([d[1] for d in dets], np.int64), g[f"dets{i}_cls"])
        np.testing.assert_array_equal(np.array([d[2] for d in dets]), g[f"dets{i}_score"])


def test_pillar_cap_is_identity_when_not_binding():
    rng = np.random.default_rng(0)
    pts = rng.uniform(0, 10, size=(500, 2)).astype(np.float32)
    flat = O.bin_points(pts, (20, 20), (0.0, 0.0), (0.5, 0.5))
    a = O.pillar_index(flat, (20, 20), 4, None)
    b = O.pillar_index(flat, (20, 20), 4, len(a.coords))
    np.testing.assert_array_equal(a.pt_idx, b.pt_idx)
    c = O.pillar_index(flat, (20, 20), 4, 10)
    assert len(c.coords) == 10
    # kept cells are those whose first point comes earliest in scene order
    firsts = {}
    for i, f in enumerate(flat):
        firsts.setdefault(int(f), i)
    want = sorted(sorted(firsts, key=lambda k: firsts[k])[:10])
    np.testing.assert_array_equal(c.coords[:, 0] * 20 + c.coords[:, 1], want)
