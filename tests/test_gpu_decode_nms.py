"""GPU decode_and_nms (K11b) against the reference's golden detections and the oracle
(pm/detector.py:266-307, pm/metrics.py:52-66).

Exactness contract: every decision (which cells are local peaks, which pass the
threshold, the stable order, which boxes survive NMS) and every class id are exact;
scores and box sizes go through exp(), where the GPU's libm and the reference's numpy
(numpy 2.3.5 dispatches f64 exp to SVML on AVX512_SKX hosts, to a Tang table method
on AVX512F ones -- different bits on different CPUs) may differ by an ulp, so those
values are compared to <= 2 ulp and the box centres, which need no exp, exactly.
"""

import json
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import pillars_oracle as O
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


def _cfg(field=16.0, base=2.5, score=0.1, iou=0.5):
    return SimpleNamespace(field_size=field, base_size=base, score_thresh=score, nms_iou=iou)


def _check(got, want_boxes, want_cls, want_scores):
    assert len(got) == len(want_cls)
    if not got:
        return
    np.testing.assert_array_equal(np.array([d.class_id for d in got], np.int64), np.asarray(want_cls, np.int64))
    boxes = np.array([d.box for d in got])
    want_boxes = np.asarray(want_boxes, np.float64).reshape(-1, 4)
    np.testing.assert_array_equal(boxes[:, :2], want_boxes[:, :2])  # centres: no exp on the path
    np.testing.assert_array_max_ulp(boxes[:, 2:], want_boxes[:, 2:], maxulp=2)
    np.testing.assert_array_max_ulp(np.array([d.score for d in got]), np.asarray(want_scores), maxulp=2)


def _oracle(cls, reg, cfg):
    dets = O.decode_and_nms(cls, reg, cfg.field_size, cfg.base_size, cfg.score_thresh, cfg.nms_iou)
    return [d[0] for d in dets], [d[1] for d in dets], [d[2] for d in dets]


def test_decode_and_nms_reference_golden(pm, golden):
    g = golden("ref_toy.npz")
    meta = json.loads((GOLDEN / "ref_toy_meta.json").read_text())
    det, dec = meta["detector"], meta["decode"]
    cfg = _cfg(det["field_size"], det["base_size"], 0.1, 0.5)
    total = 0
    for i in range(meta["n_samples"]):
        got = pm.decode_and_nms(g[f"out_FP32_{i}_cls"], g[f"out_FP32_{i}_reg"], cfg,
                                score_thresh=dec["score_thresh"], iou_thresh=dec["iou_thresh"])
        _check(got, g[f"dets{i}_box"], g[f"dets{i}_cls"], g[f"dets{i}_score"])
        total += len(got)
    assert total > 0


@pytest.mark.parametrize("shape,score,iou,seed", [((3, 8, 8), 0.05, 0.3, 0), ((3, 64, 48), 0.2, 0.5, 1),
                                                  ((2, 128, 128), 0.6, 0.1, 2), ((1, 1, 1), 0.0, 0.0, 3),
                                                  ((4, 5, 37), 1.0, 1.0, 4), ((2, 40, 30), 0.0, 0.7, 5)])
def test_decode_and_nms_vs_oracle(pm, shape, score, iou, seed):
    rng = np.random.default_rng(seed)
    C, H, W = shape
    cls = rng.normal(scale=2.0, size=(1, C, H, W)).astype(np.float32)
    reg = rng.normal(scale=1.5, size=(1, 4, H, W)).astype(np.float32)
    cfg = _cfg(field=float(max(H, W)), base=2.0, score=score, iou=iou)
    got = pm.decode_and_nms(cls, reg, cfg)
    _check(got, *_oracle(cls, reg, cfg))


def test_decode_and_nms_ties_plateaus_and_nan(pm):
    """Equal scores (plateaus: every cell a peak, order by cell index), saturated
    logits (distinct logits, identical f64 scores 1.0), NaN logits (never a peak, and
    no neighbour of a NaN is one), clipped size deltas and NaN deltas."""
    rng = np.random.default_rng(9)
    C, H, W = 3, 24, 20
    cls = rng.normal(size=(1, C, H, W)).astype(np.float32)
    cls[0, 0, 2:10, 3:12] = 1.25                 # plateau
    cls[0, 1, 5:9, 5:9] = np.float32(40.0)       # sigmoid == 1.0 exactly
    cls[0, 1, 6, 6] = np.float32(45.0)
    cls[0, 2, 10, 10] = np.nan
    cls[0, 2, 0, 0] = np.nan
    reg = rng.normal(scale=3.0, size=(1, 4, H, W)).astype(np.float32)
    reg[0, 2, 3, 4] = 9.0                        # clipped at +4
    reg[0, 3, 7, 7] = -9.0                       # clipped at -4
    reg[0, 2, 8, 8] = np.nan                     # Python's max(-4.0, nan) -> -4.0
    for score, iou in ((0.0, 0.5), (0.3, 0.0), (0.5, 1.0)):
        cfg = _cfg(field=24.0, base=1.5, score=score, iou=iou)
        got = pm.decode_and_nms(cls, reg, cfg)
        _check(got, *_oracle(cls, reg, cfg))


def test_decode_and_nms_batch_and_limits(pm):
    rng = np.random.default_rng(3)
    B, C, H, W = 5, 3, 16, 12
    cls = rng.normal(scale=2.0, size=(B, C, H, W)).astype(np.float32)
    reg = rng.normal(size=(B, 4, H, W)).astype(np.float32)
    cfg = _cfg(field=16.0, score=0.2, iou=0.4)
    dets, n = pm.decode_and_nms_batch(cls, reg, cfg)
    dets, n = dets.cpu().numpy(), n.cpu().numpy()
    for b in range(B):
        one = pm.decode_and_nms(cls[b], reg[b], cfg)
        flat = np.concatenate([dets[b, c, : n[b, c]] for c in range(C)])
        assert len(one) == len(flat)
        np.testing.assert_array_equal(np.array([d.box for d in one]).reshape(-1, 4), flat[:, :4])
        np.testing.assert_array_equal(np.array([d.score for d in one]), flat[:, 4])
    with pytest.raises(ValueError, match=r"thresholds must lie in \[0, 1\]"):
        pm.decode_and_nms(cls[0], reg[0], cfg, score_thresh=1.5)
    with pytest.raises(ValueError, match=r"thresholds must lie in \[0, 1\]"):
        pm.decode_and_nms(cls[0], reg[0], cfg, iou_thresh=-0.1)
    big = rng.normal(size=(1, 1, 129, 128)).astype(np.float32)
    with pytest.raises(RuntimeError, match="16384 cells"):
        pm.decode_and_nms(big, np.zeros((1, 4, 129, 128), np.float32), cfg)
