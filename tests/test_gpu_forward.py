"""Forward / calibration / engine parity (tiers T1, T2 of SURVEY §8(d)).

* toy detector (the reference's own model) through the drop-in ``forward`` vs the
  reference's golden outputs;
* INT8 integer accumulators bit-exact (identity scales, integer data);
* per-layer teacher-forced outputs vs the oracle (<= 1e-5 rel L2);
* KITTI-shaped PointPillars end to end (points -> heads -> top-k) vs the oracle,
  FP32 <= 1e-4, mixed/INT8 <= 1e-2 relative L2 per head;
* GPU calibration vs the reference's calibration;
* CUDA-graph replay and batching are bit-identical to eager single-frame runs.
"""

import json

import numpy as np
import pytest

from oracle import pillars_oracle as O
from tests.conftest import GOLDEN
from tests.test_oracle_golden import PLANS, _precisions, toy_stats

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _plan(pm, pname):
    return {"FP32": pm.PrecisionPlan(), "INT8": pm.PrecisionPlan(default=pm.DType.INT8),
            "FP16": pm.PrecisionPlan(default=pm.DType.FP16),
            "FP16_1_12_3": pm.parse_plan_label("FP16: 1,12,3")}[pname]


@pytest.mark.parametrize("pname,tol", [("FP32", 1e-5), ("FP16", 2e-3), ("INT8", 1e-2), ("FP16_1_12_3", 1e-2)])
def test_toy_forward_vs_reference_golden(pm, golden, pname, tol):
    g = golden("ref_toy.npz")
    graph = pm.load_model(GOLDEN / "toy")
    stats = toy_stats(g, graph)
    planned = pm.apply_plan(pm.fold_all_bn(graph), _plan(pm, pname))
    n = json.loads((GOLDEN / "ref_toy_meta.json").read_text())["n_samples"]
    for i in range(n):
        sample = pm.PillarSample(g[f"feat{i}"], g[f"mask{i}"], g[f"coords{i}"], (16, 16))
        cls_map, reg_map = pm.forward(planned, sample, stats=stats)
        assert cls_map.shape == g[f"out_{pname}_{i}_cls"].shape
        assert rel_l2(cls_map, g[f"out_{pname}_{i}_cls"]) <= tol
        assert rel_l2(reg_map, g[f"out_{pname}_{i}_reg"]) <= tol


def test_toy_unfolded_bn_forward(pm, golden):
    g = golden("ref_toy.npz")
    graph = pm.load_model(GOLDEN / "toy")
    for i in range(3):
        sample = pm.PillarSample(g[f"feat{i}"], g[f"mask{i}"], g[f"coords{i}"], (16, 16))
        c, r = pm.forward(graph, sample)
        assert rel_l2(c, g[f"out_UNFOLDED_{i}_cls"]) <= 1e-5
        assert rel_l2(r, g[f"out_UNFOLDED_{i}_reg"]) <= 1e-5


def test_forward_errors_match_reference(pm):
    rng = np.random.default_rng(13)
    layers = (pm.LayerSpec(name="lin1", kind="linear", index=1, weight=rng.normal(size=(6, 6)).astype(np.float32),
                           bias=np.zeros(6, np.float32), relu=True),
              pm.LayerSpec(name="lin2", kind="linear", index=2, weight=rng.normal(size=(4, 6)).astype(np.float32),
                           bias=np.zeros(4, np.float32)))
    g = pm.ModelGraph(layers=layers)
    q = pm.apply_plan(g, pm.PrecisionPlan(default=pm.DType.INT8))
    with pytest.raises(RuntimeError, match="layer 1 .*'lin1'.* no quant params"):
        pm.forward(q, np.zeros((1, 6), np.float32))
    x = rng.normal(size=(3, 6)).astype(np.float32)
    want = O.linear(O.relu(O.linear(x, layers[0].weight, layers[0].bias)), layers[1].weight, layers[1].bias)
    assert rel_l2(pm.forward(g, x), want) < 1e-6
    stats = pm.run_calibration(g, [np.zeros((2, 6), np.float32)])
    assert stats[1].act_qp.scale == 1.0
    q1 = pm.apply_plan(g, pm.PrecisionPlan(overrides={1: pm.DType.INT8}))
    np.testing.assert_array_equal(pm.forward(q1, np.zeros((2, 6), np.float32), stats=stats),
                                  pm.forward(g, np.zeros((2, 6), np.float32)))


def test_observe_fn_sees_pre_transform_inputs(pm, golden):
    g = golden("ref_toy.npz")
    graph = pm.fold_all_bn(pm.load_model(GOLDEN / "toy"))
    sample = pm.PillarSample(g["feat0"], g["mask0"], g["coords0"], (16, 16))
    seen_gpu, seen_cpu = {}, {}
    pm.forward(graph, sample, observe_fn=lambda l, x: seen_gpu.__setitem__(l.index, np.array(x)))
    O.forward(graph, O.Sample(g["feat0"], g["mask0"], g["coords0"], (16, 16)),
              observe_fn=lambda l, x: seen_cpu.__setitem__(l.index, np.array(x)))
    assert sorted(seen_gpu) == sorted(seen_cpu)
    for i in seen_cpu:
        assert seen_gpu[i].shape == seen_cpu[i].shape, i
        assert rel_l2(seen_gpu[i], seen_cpu[i]) <= 1e-5, i


def test_gpu_calibration_vs_reference(pm, golden):
    g = golden("ref_toy.npz")
    graph = pm.load_model(GOLDEN / "toy")
    samples = [pm.PillarSample(g[f"feat{i}"], g[f"mask{i}"], g[f"coords{i}"], (16, 16)) for i in range(4)]
    st = pm.run_calibration(graph, samples, per_channel_weights=True)
    for l in graph.weight_layers:
        i = l.index
        lo, hi = g[f"stat{i}_minmax"]
        assert st[i].observer.running_min == pytest.approx(lo, rel=1e-5, abs=1e-6)
        assert st[i].observer.running_max == pytest.approx(hi, rel=1e-5, abs=1e-6)
        assert st[i].act_qp.scale == pytest.approx(float(g[f"stat{i}_act"]), rel=1e-5)
        np.testing.assert_array_equal(st[i].weight_qp.scales, g[f"statpc{i}_w"])
        assert st[i].observer.count == 4
    bad = pm.PillarSample(np.full_like(g["feat1"], np.inf), g["mask1"], g["coords1"], (16, 16))
    with pytest.raises(RuntimeError, match="layer 1 .* sample 1"):
        pm.run_calibration(graph, [samples[0], bad])


# ----------------------------------------------------------------------------- integer accumulators


@pytest.mark.parametrize("cin,cout,k,stride,hw", [(64, 64, 3, 2, (20, 18)), (128, 256, 3, 1, (9, 7)),
                                                  (64, 128, 1, 1, (5, 6)), (256, 128, 4, 4, (3, 4)),
                                                  (384, 20, 1, 1, (6, 5))])
def test_int8_accumulators_exact(pm, cin, cout, k, stride, hw):
    """Integer-valued inputs/weights with unit scales: y == float(sum of int products) exactly."""
    rng = np.random.default_rng(cin + cout + k)
    x = rng.integers(-127, 128, size=(2, cin) + hw).astype(np.float32)
    w = rng.integers(-127, 128, size=(cout, cin, k, k)).astype(np.float32)
    deconv = k == stride and k > 1
    layer = pm.LayerSpec(name="l", kind="deconv2d" if deconv else "conv2d", index=1, weight=w,
                         bias=np.zeros(cout, np.float32),
                         conv=pm.ConvParams(stride=(stride, stride), padding=(0, 0) if deconv or k == 1 else (1, 1)))
    g = pm.apply_plan(pm.ModelGraph(layers=(layer,)), pm.PrecisionPlan(default=pm.DType.INT8))
    stats = O.Stats(layers={1: O.LayerStats(1, "l", O._Obs(-127, 127, 1), O._QP(1.0), O._QP(1.0))})
    got = pm.forward(g, x, stats=stats)
    xi, wi = x.astype(np.int64), w.astype(np.int64)
    if deconv:
        want = O.deconv2d(x.astype(np.float64), w.astype(np.float64), np.zeros(cout), (k, k))
    else:
        want = O.conv2d(x.astype(np.float64), w.astype(np.float64), np.zeros(cout), (stride, stride),
                        (0, 0) if k == 1 else (1, 1))
    assert np.abs(want).max() < 2 ** 24
    np.testing.assert_array_equal(got, want.astype(np.float32))
    del xi, wi


# ----------------------------------------------------------------------------- teacher-forced layers


@pytest.mark.parametrize("prec", ["fp32", "fp16", "int8"])
@pytest.mark.parametrize("kind", ["conv_s2", "conv_s1", "deconv2", "deconv4", "head"])
def test_teacher_forced_layer(pm, prec, kind):
    rng = np.random.default_rng(hash((prec, kind)) % 2 ** 32)
    spec = {"conv_s2": (64, 64, 3, 2, (24, 20)), "conv_s1": (128, 128, 3, 1, (12, 10)),
            "deconv2": (128, 128, 2, 2, (6, 5)), "deconv4": (256, 128, 4, 4, (3, 3)),
            "head": (384, 14, 1, 1, (12, 10))}[kind]
    cin, cout, k, s, hw = spec
    x = np.maximum(rng.normal(size=(1, cin) + hw), 0).astype(np.float32)
    w = rng.normal(scale=np.sqrt(2.0 / (cin * k * k)), size=(cout, cin, k, k)).astype(np.float32)
    b = rng.normal(scale=0.1, size=cout).astype(np.float32)
    deconv = kind.startswith("deconv")
    layer = pm.LayerSpec(name="l", kind="deconv2d" if deconv else "conv2d", index=1, weight=w, bias=b,
                         relu=kind != "head",
                         conv=pm.ConvParams(stride=(s, s), padding=(0, 0) if (deconv or k == 1) else (1, 1)))
    graph = pm.ModelGraph(layers=(layer,))
    st = pm.run_calibration(graph, [x], per_channel_weights=True)
    planned = pm.apply_plan(graph, pm.PrecisionPlan(default=pm.DType(prec)))
    got = pm.forward(planned, x, stats=st)
    want = O.run_weight_layer(planned.layers[0], x, st)
    assert rel_l2(got, want) <= 1e-5


# ----------------------------------------------------------------------------- KITTI end to end


def _oracle_e2e(pm, graph, cfg, frame, stats, plan, acc=np.float32):
    folded = pm.fold_all_bn(graph)
    planned = pm.apply_plan(folded, plan)
    sample, _ = O.pillarize_kitti(frame, cfg.grid_spec())
    precs = {l.index: l.precision.value for l in planned.weight_layers}
    with O.accumulate_in(acc):
        return O.forward(O.folded_graph(planned, precs), sample, stats=stats)


# T2 protocol: every implementation that does not replicate
# OpenBLAS's summation order bit for bit flips near-tie INT8 codes, and the flips
# cascade.  The bar is therefore: FP32 <= 1e-4 and FP16 <= 1e-2 absolutely; plans
# with INT8 layers <= max(1e-2, 2 x the reference's own re-association noise floor
# |ref_f32 - ref_f64|), and for all-INT8 (exact int32 accumulation) the engine must
# equal the f64-accumulated reference semantics to 1e-5.
@pytest.mark.parametrize("label", ["FP32", "FP16", "FP16: 2,18,19,20", "INT8", "FP16: 1,22,3"])
def test_kitti_small_end_to_end(pm, label):
    cfg = pm.PointPillarsConfig.small(max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=1)
    calib = [pm.make_frame(3000, 100 + i, cfg, outlier_frac=0.01) for i in range(2)]
    ranges = O.per_sample_ranges(graph, [O.pillarize_kitti(f, cfg.grid_spec())[0] for f in calib])
    stats = pm.calibration.stats_from_ranges(graph, ranges, per_channel_weights=True)
    frame = pm.make_frame(3000, 7, cfg)
    plan = pm.parse_plan_label(label)
    eng = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=1, max_points_per_frame=4000)
    eng.load_points([frame])
    eng.run()
    heads = {k: v.cpu().numpy() for k, v in eng.heads_nchw().items()}
    ref32 = _oracle_e2e(pm, graph, cfg, frame, stats, plan)
    ref64 = _oracle_e2e(pm, graph, cfg, frame, stats, plan, np.float64)
    refint = _oracle_e2e(pm, graph, cfg, frame, stats, plan, "int")
    for name, r32, r64, ri in zip(pm.pointpillars.HEADS, ref32, ref64, refint):
        err = rel_l2(heads[name][0], r32[0])
        if label == "FP32":
            assert err <= 1e-4, (label, name, err)
        elif label == "FP16":
            assert err <= 1e-2, (label, name, err)
        else:
            # noise floor: how far two valid executions of the same plan drift apart
            floor = max(rel_l2(r32[0], r64[0]), rel_l2(r32[0], ri[0]))
            assert err <= max(1e-2, 2 * floor), (label, name, err, floor)
        if label == "INT8":  # exact int32 accumulation == the integer-execution semantics
            assert rel_l2(heads[name][0], ri[0]) <= 1e-5, (name, rel_l2(heads[name][0], ri[0]))
        elif label not in ("FP32", "FP16"):
            # mixed plans: a fixed bar against the integer-execution semantics (INT8 layers
            # exact; the FP16 layers' f32 accumulation order is the only difference)
            assert rel_l2(heads[name][0], ri[0]) <= 2e-4, (label, name, rel_l2(heads[name][0], ri[0]))


def test_engine_calibration_matches_oracle(pm):
    cfg = pm.PointPillarsConfig.small(max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=2)
    frames = [pm.make_frame(3000, 200 + i, cfg, outlier_frac=0.01) for i in range(2)]
    st, ranges = pm.calibrate_frames(graph, frames, cfg, return_ranges=True)
    want = O.per_sample_ranges(graph, [O.pillarize_kitti(f, cfg.grid_spec())[0] for f in frames])
    for r, w in zip(ranges, want):
        assert set(r) == set(w)
        assert r[1] == w[1]  # layer-1 input (the 9 pillar features) is bit-exact
        for i in w:
            np.testing.assert_allclose(r[i], w[i], rtol=1e-5, atol=1e-6)


def test_graph_replay_and_batch_are_bit_identical(pm):
    cfg = pm.PointPillarsConfig.small(max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=3)
    frames = [pm.make_frame(2500 + 300 * i, 300 + i, cfg) for i in range(3)]
    stats = pm.calibrate_frames(graph, frames[:2], cfg)
    single = []
    for f in frames:
        e = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=1, max_points_per_frame=4000)
        e.load_points([f])
        e.run()
        single.append(({k: v.clone() for k, v in e.heads().items()}, {k: v.clone() for k, v in e.topk().items()}))
    eb = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=3, max_points_per_frame=4000)
    eb.capture()
    eb.load_points(frames)
    eb.run()
    eb.run()
    for b, (h1, t1) in enumerate(single):
        for k in h1:
            assert (eb.heads()[k][b] == h1[k][0]).all(), k
        for k in t1:
            assert (eb.topk()[k][b] == t1[k][0]).all(), k


@pytest.mark.slow
def test_kitti_full_size_fp32_vs_oracle(pm):
    cfg = pm.PointPillarsConfig()
    graph = pm.build_pointpillars(cfg, seed=0)
    frame = pm.make_frame(20000, 1, cfg)
    eng = pm.PointPillarsEngine(graph, "FP32", None, cfg, batch=1, max_points_per_frame=20000)
    eng.load_points([frame])
    eng.run()
    heads = {k: v.cpu().numpy() for k, v in eng.heads_nchw().items()}
    want = _oracle_e2e(pm, graph, cfg, frame, None, pm.PrecisionPlan())
    for name, ref in zip(pm.pointpillars.HEADS, want):
        assert rel_l2(heads[name][0], ref[0]) <= 1e-4, name


def test_pipelined_engine_matches_sequential(pm):
    """PipelinedEngine (double-buffered H2D / graph / D2H streaming) returns, for every
    batch, exactly the records of running that batch alone."""
    import torch

    from paper_2601_12638_b200 import distributed as D

    cfg = pm.PointPillarsConfig.small(max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=4)
    stats = pm.calibrate_frames(graph, [pm.make_frame(3000, 400 + i, cfg) for i in range(2)], cfg)
    batches_np = [[pm.make_frame(2000 + 500 * j + 100 * i, 500 + 10 * j + i, cfg) for i in range(2)] for j in range(5)]
    want = []
    for fr in batches_np:
        e = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=2, max_points_per_frame=5000)
        e.load_points(fr)
        e.run()
        want.append(D.pack_topk(e.topk()).cpu())
        # the in-graph records op (pmx_pack_topk_records) == the torch packing, bit for bit
        assert torch.equal(e.cg.records.cpu(), want[-1])
    eng = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=2, max_points_per_frame=5000)
    eng.load_points(batches_np[0])
    pipe = pm.PipelinedEngine(eng)
    batches = []
    for fr in batches_np:
        offs = np.zeros(3, np.int64)
        offs[1:] = np.cumsum([len(f) for f in fr])
        batches.append((torch.from_numpy(np.concatenate(fr)).pin_memory(), torch.from_numpy(offs).pin_memory()))
    outs = [torch.empty_like(w).pin_memory() for w in want]
    pipe.run(batches, outs, D.pack_topk)
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert torch.equal(o, w)
    # default: the records each slot's graph wrote, read back without extra kernels
    outs2 = [torch.empty_like(w).pin_memory() for w in want]
    pipe.run(batches, outs2)
    torch.cuda.synchronize()
    for o, w in zip(outs2, want):
        assert torch.equal(o, w)


def test_pipelined_engine_split_graphs_two_engines(pm):
    """Batch 9 (no side-stream branches): each slot replays two graphs (pillarize + PFN,
    then the rest) and the next H2D into a slot waits only for the first; two engines
    alternate on their own streams.  Every batch's records equal its sequential run."""
    import torch

    from paper_2601_12638_b200 import distributed as D

    cfg = pm.PointPillarsConfig.small(max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=6)
    stats = pm.calibrate_frames(graph, [pm.make_frame(3000, 800 + i, cfg) for i in range(2)], cfg)
    B = 9
    batches_np = [[pm.make_frame(1500 + 100 * i + 37 * j, 900 + 10 * j + i, cfg) for i in range(B)] for j in range(7)]
    ref = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=B, max_points_per_frame=3000)
    want = []
    for fr in batches_np:
        ref.load_points(fr)
        ref.run()
        want.append(D.pack_topk(ref.topk()).cpu())
    e1 = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=B, max_points_per_frame=3000)
    e2 = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=B, max_points_per_frame=3000)
    e1.load_points(batches_np[0])
    e2.load_points(batches_np[0])
    pipe = pm.PipelinedEngine(e1, e2)
    assert all(sp is not None for sp in pipe.split)
    batches = []
    for fr in batches_np:
        offs = np.zeros(B + 1, np.int64)
        offs[1:] = np.cumsum([len(f) for f in fr])
        batches.append((torch.from_numpy(np.concatenate(fr)).pin_memory(), torch.from_numpy(offs).pin_memory()))
    outs = [torch.empty_like(w).pin_memory() for w in want]
    pipe.run(batches, outs)
    torch.cuda.synchronize()
    for j, (o, w) in enumerate(zip(outs, want)):
        assert torch.equal(o, w), j


def test_pipelined_engine_batch1_many_distinct_frames(pm):
    """Batch 1 (short graphs) over many distinct frames: every slot's records buffer is
    rewritten only after the previous D2H copy of that slot finished (no WAR race)."""
    import torch

    from paper_2601_12638_b200 import distributed as D

    cfg = pm.PointPillarsConfig.small(max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=5)
    stats = pm.calibrate_frames(graph, [pm.make_frame(3000, 600 + i, cfg) for i in range(2)], cfg)
    frames = [pm.make_frame(1500 + 37 * j, 700 + j, cfg) for j in range(24)]
    eng = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=1, max_points_per_frame=3000)
    want = []
    for f in frames:
        eng.load_points([f])
        eng.run()
        want.append(D.pack_topk(eng.topk()).cpu())
    pipe = pm.PipelinedEngine(eng)
    batches = [(torch.from_numpy(f).pin_memory(), torch.from_numpy(np.array([0, len(f)], np.int64)).pin_memory())
               for f in frames]
    for _ in range(3):
        outs = [torch.empty_like(w).pin_memory() for w in want]
        pipe.run(batches, outs)
        torch.cuda.synchronize()
        for j, (o, w) in enumerate(zip(outs, want)):
            assert torch.equal(o, w), j


def test_pipelined_two_engines_match_sequential(pm):
    """PipelinedEngine over two engine instances (own buffers, one compute stream each:
    consecutive batches overlap on the SMs) returns every batch's own records."""
    import torch

    from paper_2601_12638_b200 import distributed as D

    cfg = pm.PointPillarsConfig.small(max_pillars=1500)
    graph = pm.build_pointpillars(cfg, seed=6)
    stats = pm.calibrate_frames(graph, [pm.make_frame(3000, 800 + i, cfg) for i in range(2)], cfg)
    batches_np = [[pm.make_frame(1800 + 90 * j + 40 * i, 900 + 10 * j + i, cfg) for i in range(2)] for j in range(9)]
    e1 = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=2, max_points_per_frame=3000)
    e2 = pm.PointPillarsEngine(graph, pm.MIXED_PLAN_LABEL, stats, cfg, batch=2, max_points_per_frame=3000)
    want = []
    for fr in batches_np:
        e1.load_points(fr)
        e1.run()
        want.append(D.pack_topk(e1.topk()).cpu())
    pipe = pm.PipelinedEngine(e1, e2)
    batches = []
    for fr in batches_np:
        offs = np.zeros(3, np.int64)
        offs[1:] = np.cumsum([len(f) for f in fr])
        batches.append((torch.from_numpy(np.concatenate(fr)).pin_memory(), torch.from_numpy(offs).pin_memory()))
    for _ in range(2):
        outs = [torch.empty_like(w).pin_memory() for w in want]
        pipe.run(batches, outs)
        torch.cuda.synchronize()
        for j, (o, w) in enumerate(zip(outs, want)):
            assert torch.equal(o, w), j


def test_int8_plan_tcgen05_equals_simt_end_to_end(pm):
    """All-INT8 plan, two full-size KITTI frames: every conv through the tcgen05 kernels
    (swizzled halos, cp.async gather, staged stores, fused heads) vs every conv through
    the SIMT kernels (dense canvas, no gather).  Integer arithmetic end to end, so the
    head maps and the top-k must be identical bit for bit."""
    import torch

    from paper_2601_12638_b200 import _native as N

    lib = N.load()
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=11)
    frames = [pm.make_frame(120000, 70 + i, cfg) for i in range(2)]
    stats = pm.calibrate_frames(graph, [pm.make_frame(120000, 80, cfg, 0.01)], cfg)
    got = {}
    for mode in (0, 1):
        lib.pmx_set_conv_backend(mode)
        try:
            e = pm.PointPillarsEngine(graph, "INT8", stats, cfg, batch=2, max_points_per_frame=120000)
            e.load_points(frames)
            e.run()
            torch.cuda.synchronize()
            got[mode] = ({k: v.clone() for k, v in e.heads().items()}, e.topk()["idx"].clone())
        finally:
            lib.pmx_set_conv_backend(0)
    for name in got[0][0]:
        assert torch.equal(got[0][0][name], got[1][0][name]), name
    assert torch.equal(got[0][1], got[1][1])
