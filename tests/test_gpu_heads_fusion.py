"""Deconvs with the three INT8 heads fused into their epilogues (pmx_deconv_heads): the
concat is never written, the heads block and the top-k are bit-identical to the
unfused deconv -> concat -> fused-heads GEMM path (int32 head partial sums are exact
and order-free; the last deconv applies the heads' own epilogue formula)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


def _run(pm, graph, plan, stats, cfg, frames, fuse):
    old = os.environ.get("PMX_FUSE_HEADS")
    os.environ["PMX_FUSE_HEADS"] = "1" if fuse else "0"
    try:
        eng = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=len(frames),
                                    max_points_per_frame=max(len(f) for f in frames))
    finally:
        if old is None:
            del os.environ["PMX_FUSE_HEADS"]
        else:
            os.environ["PMX_FUSE_HEADS"] = old
    eng.load_points(frames)
    eng.run()
    return eng, eng.cg.heads_cat.clone(), {k: v.clone() for k, v in eng.topk().items()}


@pytest.mark.parametrize("size", ["small", "full"])
@pytest.mark.parametrize("label", ["INT8", "FP16: 2,18,19,20", "FP16: 1,22,3"])
def test_fused_heads_bit_identical(pm, size, label):
    import torch

    if size == "full":
        cfg = pm.PointPillarsConfig(max_pillars=16000)
        frames = [pm.make_frame(120000, 41 + i, cfg) for i in range(2)]
        calib = [pm.make_frame(120000, 51, cfg, 0.01)]
    else:
        cfg = pm.PointPillarsConfig.small(grid=(96, 80), max_pillars=2500)
        frames = [pm.make_frame(4000 + 700 * i, 41 + i, cfg) for i in range(3)]
        calib = [pm.make_frame(4000, 51, cfg, 0.01)]
    graph = pm.build_pointpillars(cfg, seed=9)
    stats = pm.calibrate_frames(graph, calib, cfg, per_channel_weights=True)
    ef, hf, tf = _run(pm, graph, label, stats, cfg, frames, True)
    eu, hu, tu = _run(pm, graph, label, stats, cfg, frames, False)
    names = [n for n, _ in ef.cg.ops]
    if label == "FP16: 1,22,3":  # head 22 in FP16: the heads' input formats differ -> no fusion
        assert ef.cg.hfuse is None and not any(n.endswith("+heads") for n in names)
    else:
        assert ef.cg.hfuse is not None and "conv heads(fused)" not in names
        assert sum(n.endswith("+heads") for n in names) == 3
    assert eu.cg.hfuse is None
    assert torch.equal(hf, hu)
    for k in tf:
        assert torch.equal(tf[k], tu[k]), k


def test_fused_heads_captured_graph_replays(pm):
    """The fused path inside a captured CUDA graph, replayed over different frames."""
    import torch

    cfg = pm.PointPillarsConfig.small(grid=(64, 48), max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=10)
    stats = pm.calibrate_frames(graph, [pm.make_frame(3000, 61, cfg)], cfg)
    batches = [[pm.make_frame(2000 + 300 * j + 50 * i, 70 + 10 * j + i, cfg) for i in range(2)] for j in range(3)]
    old = os.environ.get("PMX_FUSE_HEADS")
    os.environ["PMX_FUSE_HEADS"] = "1"
    try:
        eng = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=2, max_points_per_frame=3000)
    finally:
        if old is None:
            del os.environ["PMX_FUSE_HEADS"]
        else:
            os.environ["PMX_FUSE_HEADS"] = old
    assert eng.cg.hfuse is not None
    eng.capture()
    for fr in batches:
        eng.load_points(fr)
        eng.run()
        got = eng.cg.heads_cat.clone()
        _, want, _ = _run(pm, graph, pm.MIXED_PLAN_LABEL, stats, cfg, fr, False)
        assert torch.equal(got, want)
