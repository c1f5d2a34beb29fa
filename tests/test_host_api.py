"""Host-side API semantics (no GPU): plans, labels, graph validation, BN folding,
serialization, calibration-set selection, stats files -- ported from the
reference's own tests (pkg/tests/test_model.py, test_calibration.py)."""

import dataclasses
import json

import numpy as np
import pytest

from paper_2601_12638_b200 import calibration as CAL
from paper_2601_12638_b200.model import (
    BatchNorm,
    LayerSpec,
    ModelFormatError,
    ModelGraph,
    PrecisionPlan,
    UnsupportedVersionError,
    apply_plan,
    dtype_boundaries,
    fold_bn,
    graphs_equal,
    load_model,
    parse_plan_label,
    save_model,
    weights_digest,
)
from paper_2601_12638_b200.pointpillars import PointPillarsConfig, build_pointpillars
from paper_2601_12638_b200.quant import (DType, MinMaxObserver, PerChannelQuantParams, QuantParams, compute_scale,
                                         weight_quant_params)
from paper_2601_12638_b200.tensor_ops import ConvParams
from tests.conftest import GOLDEN


def lin(index, din, dout, rng, bn=None, relu=False):
    return LayerSpec(name=f"lin{index}", kind="linear", index=index,
                     weight=rng.normal(scale=0.5, size=(dout, din)).astype(np.float32),
                     bias=rng.normal(scale=0.1, size=dout).astype(np.float32), bn=bn, relu=relu)


def rbn(c, rng, eps=1e-5):
    return BatchNorm(gamma=rng.uniform(0.5, 1.5, c).astype(np.float32), beta=rng.normal(scale=0.2, size=c).astype(np.float32),
                     mean=rng.normal(scale=0.3, size=c).astype(np.float32), var=rng.uniform(0.5, 2.0, c).astype(np.float32),
                     eps=eps)


def test_compute_scale_examples():
    assert compute_scale(-1.0, 2.0).scale == 2.0 / 127.0
    assert compute_scale(-127.0, 127.0).scale == 1.0
    assert compute_scale(0.0, 0.0).scale == 1.0
    with pytest.raises(ValueError, match="non-finite"):
        compute_scale(-np.inf, 1.0)
    with pytest.raises(ValueError, match="min .* > max"):
        compute_scale(2.0, 1.0)
    with pytest.raises(ValueError, match="positive"):
        QuantParams(scale=0.0)
    with pytest.raises(ValueError, match="zero_point"):
        QuantParams(scale=1.0, zero_point=3)


def test_plan_labels():
    plan = parse_plan_label("FP16: 1,22,3")
    assert list(plan.overrides) == [1, 22, 3]
    assert plan.label() == "FP16: 1,22,3"
    assert parse_plan_label("int8").default is DType.INT8
    with pytest.raises(ValueError, match="unrecognized"):
        parse_plan_label("FP8")
    rng = np.random.default_rng(6)
    g = ModelGraph(layers=tuple(lin(i, 4, 4, rng) for i in range(1, 24)))
    out = apply_plan(g, parse_plan_label("FP16: 1,22"))
    tags = {l.index: l.precision for l in out.weight_layers}
    assert tags[1] is DType.FP16 and tags[22] is DType.FP16 and tags[2] is DType.INT8
    with pytest.raises(ValueError, match=r"unknown layer indices \[99\]"):
        apply_plan(g, PrecisionPlan(overrides={99: DType.FP16}))
    digest = weights_digest(g)
    apply_plan(g, PrecisionPlan(default=DType.INT8))
    assert weights_digest(g) == digest
    fp16, int8 = DType.FP16, DType.INT8
    assert dtype_boundaries([fp16] + [int8] * 20 + [fp16, int8]) == 3


def test_graph_validation():
    rng = np.random.default_rng(15)
    with pytest.raises(ValueError, match="expected 1"):
        ModelGraph(layers=(lin(2, 3, 3, rng),))
    with pytest.raises(ValueError, match="unknown kind"):
        ModelGraph(layers=(LayerSpec(name="x", kind="softmax"),))
    head = dataclasses.replace(lin(1, 3, 3, rng), is_head=True)
    with pytest.raises(ValueError, match="follows a head"):
        ModelGraph(layers=(head, lin(2, 3, 3, rng)))
    with pytest.raises(ValueError, match="unknown or later"):
        ModelGraph(layers=(lin(1, 3, 3, rng), LayerSpec(name="c", kind="concat", inputs=("nope",))))


def test_fold_bn_matches_reference_formula():
    rng = np.random.default_rng(2)
    layer = lin(1, 5, 3, rng, bn=rbn(3, rng))
    f = fold_bn(layer)
    bn = layer.bn
    factor = (bn.gamma.astype(np.float64) / np.sqrt(bn.var.astype(np.float64) + bn.eps)).astype(np.float32)
    np.testing.assert_array_equal(f.weight, (layer.weight * factor[:, None]).astype(np.float32))
    np.testing.assert_array_equal(f.bias, ((layer.bias - bn.mean) * factor + bn.beta).astype(np.float32))
    with pytest.raises(ValueError, match="no batch norm"):
        fold_bn(lin(1, 4, 3, rng))
    bad = dataclasses.replace(layer, bn=dataclasses.replace(bn, var=np.array([-1.0, 1, 1], np.float32), eps=0.0))
    with pytest.raises(ValueError, match="non-positive"):
        fold_bn(bad)


def test_serialization_round_trip(tmp_path):
    g = build_pointpillars(PointPillarsConfig.small(), seed=3)
    save_model(g, tmp_path / "pp")
    assert graphs_equal(g, load_model(tmp_path / "pp"))
    blob = bytearray((tmp_path / "pp.mpq.bin").read_bytes())
    blob[0] ^= 0xFF
    (tmp_path / "pp.mpq.bin").write_bytes(bytes(blob))
    with pytest.raises(ModelFormatError, match="checksum"):
        load_model(tmp_path / "pp")
    (tmp_path / "pp.mpq.bin").write_bytes(bytes(blob[:-8]))
    with pytest.raises(ModelFormatError, match="size"):
        load_model(tmp_path / "pp")
    doc = json.loads((tmp_path / "pp.mpq.json").read_text())
    doc["format_version"] = 99
    (tmp_path / "pp.mpq.json").write_text(json.dumps(doc))
    with pytest.raises(UnsupportedVersionError, match="99"):
        load_model(tmp_path / "pp")
    (tmp_path / "pp.mpq.json").write_text("{not json")
    with pytest.raises(ModelFormatError, match="malformed"):
        load_model(tmp_path / "pp")


def test_reads_reference_model_file():
    g = load_model(GOLDEN / "toy")
    assert g.num_indexed == 13
    assert [l.kind for l in g.layers[:3]] == ["linear", "maxpool", "scatter"]


def test_select_calib_set():
    assert sorted(CAL.select_calib_set(10, n=10, seed=3).indices) == list(range(10))
    assert CAL.select_calib_set(100, n=4, seed=9).indices == CAL.select_calib_set(100, n=4, seed=9).indices
    assert CAL.select_calib_set(200, n=64, seed=5, nested=True).indices[:4] == \
        CAL.select_calib_set(200, n=4, seed=5, nested=True).indices
    with pytest.raises(ValueError, match="out of range"):
        CAL.select_calib_set(10, n=11)


def test_stats_from_ranges_and_io(tmp_path):
    rng = np.random.default_rng(4)
    g = ModelGraph(layers=(lin(1, 6, 6, rng, relu=True), lin(2, 6, 4, rng)))
    ranges = [{1: (-1.0, 2.0), 2: (0.0, 3.0)}, {1: (-3.0, 1.0), 2: (0.0, 0.5)}]
    st = CAL.stats_from_ranges(g, ranges, seed=7, per_channel_weights=True)
    assert st[1].observer == MinMaxObserver(-3.0, 2.0, 2)
    assert st[1].act_qp.scale == 3.0 / 127.0
    np.testing.assert_array_equal(st[2].weight_qp.scales, weight_quant_params(g.layers[1].weight, True).scales)
    CAL.save_stats(st, tmp_path / "s.json")
    back = CAL.load_stats(tmp_path / "s.json")
    assert back[1].observer == st[1].observer and back[2].act_qp == st[2].act_qp
    np.testing.assert_array_equal(back[2].weight_qp.scales, st[2].weight_qp.scales)
    with pytest.raises(ValueError, match="at least one sample"):
        CAL.stats_from_ranges(g, [])


def test_pointpillars_graph_shape():
    g = build_pointpillars()
    assert g.num_indexed == 23
    names = {l.index: l.name for l in g.weight_layers}
    assert names[1] == "voxel_encoder.pfn_layers.0.linear"
    assert names[2] == "backbone.blocks.0.0" and names[17] == "backbone.blocks.2.15"
    assert names[18] == "neck.deblocks.0.0" and names[20] == "neck.deblocks.2.0"
    assert names[21] == "bbox_head.conv_dir_cls" and names[22] == "bbox_head.conv_reg"
    assert names[23] == "bbox_head.conv_cls"
    cfg = PointPillarsConfig()
    assert cfg.out_grid == (248, 216)
    assert abs(cfg.out_stride[0] - 0.32) < 1e-9


def test_sweep_ranking_and_greedy_plans():
    """Config-5 host logic: most sensitive first, ties to the lower
    index; greedy candidates are FP16 on the top-i layers over an INT8 base."""
    from paper_2601_12638_b200.sweep import greedy_candidates, head_error, records, select_topk

    errs = {1: 0.5, 2: 0.9, 3: 0.1, 4: 0.9, 5: 0.7}
    assert select_topk(errs, 5) == [2, 4, 5, 1, 3]
    assert select_topk(errs, 2) == [2, 4]
    with pytest.raises(ValueError):
        select_topk(errs, 0)
    with pytest.raises(ValueError):
        select_topk(errs, 6)
    cands = greedy_candidates([2, 4, 5], 3)
    assert [c.label() for c in cands] == ["FP16: 2", "FP16: 2,4", "FP16: 2,4,5"]
    assert cands[2].resolve(4) is DType.FP16 and cands[2].resolve(1) is DType.INT8
    assert head_error([4.0, 16.0]) == 0.5 and head_error([1.0, 0.0]) == float("inf")
    recs = records({"layer_errors": errs, "ranking": select_topk(errs, 5)})
    assert [(r.layer_index, r.rank) for r in recs] == [(1, 4), (2, 1), (3, 5), (4, 2), (5, 3)]


def test_qat_config_and_golden_stats():
    """QAT host pieces (pm/qat.py:34-64): config validation, and the reference-written
    calibration stats of the QAT fixtures load through this package's reader."""
    from paper_2601_12638_b200 import qat

    cfg = qat.TrainConfig()
    assert (cfg.learning_rate, cfg.epochs, cfg.batch_size, cfg.pos_weight) == (2e-4, 1, 4, 4.0)
    with pytest.raises(ValueError, match="learning_rate must be positive"):
        qat.TrainConfig(learning_rate=0.0)
    with pytest.raises(ValueError, match="epochs must be >= 1"):
        qat.TrainConfig(epochs=0)
    with pytest.raises(ValueError, match=r"momentum must lie in \[0, 1\)"):
        qat.TrainConfig(momentum=1.0)
    st = CAL.load_stats(GOLDEN / "qat_stats_pc.json")
    assert st.indices() == list(range(1, 14))
    assert all(isinstance(st[i].weight_qp, PerChannelQuantParams) for i in st.indices())
    g = load_model(GOLDEN / "qat_chain")
    assert [l.kind for l in g.layers] == ["conv2d", "conv2d", "upsample2x", "conv2d"]
