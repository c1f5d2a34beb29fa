"""Headline-configuration parity at BASELINE shapes (SURVEY §8(d) tiers T1 and T2).

Config 2 (all-INT8, per-channel weights, 4 calibration frames with 1% outliers) and
config 3 (mixed "FP16: 2,18,19,20", 2 calibration frames), 120k-point frames on the
full 496 x 432 grid with the 16000-pillar cap -- the frames bench.py measures.
Calibration stats come from the CPU oracle (the reference algorithm), so engine and
oracle run with identical weights, scales and pillar features.

T2 (end to end, points -> heads -> top-k):
  * engine == the oracle's integer-execution semantics (``accumulate_in("int")``:
    exact int32 accumulation of INT8 codes, one f32 rounding of acc * alpha + bias)
    -- bit-exact for the all-INT8 plan, rel L2 <= 2e-4 for the mixed plan (its FP16
    layers sum in f32 in another order than the oracle's f64);
  * engine vs the f32 reference <= max(1e-2, 1.1 x the reference's own
    re-association floor |ref_f32 - ref_f64|), the floor printed;
  * top-k anchor index set == the integer oracle's.
T1 (teacher-forced, every layer of both plans): the oracle's own input of layer l
is fed to engine layer l at its full shape; for INT8 layers the f32 output equals
the integer oracle bit for bit and every consumer buffer the production epilogue
writes (int8 codes at the consumer's scale, binary16 for an FP16 consumer) equals
quantize(y, s) / fp16_roundtrip(y) of that output exactly (flip rate 0); FP16 layers
are within 1e-5 of the f64-accumulated oracle.  Rates against the f32 reference
are printed.
"""

import dataclasses

import numpy as np
import pytest

from oracle import pillars_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N_POINTS = 120000
MAX_PILLARS = 16000
PLANS = {"C2": ("INT8", 4), "C3": ("FP16: 2,18,19,20", 2)}


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


@pytest.fixture(scope="module")
def setup(pm):
    """Per config: graph, oracle stats, one evaluation frame and its oracle runs."""
    cfg = pm.PointPillarsConfig(max_pillars=MAX_PILLARS)
    graph = pm.build_pointpillars(cfg, seed=0)
    frame = pm.make_frame(N_POINTS, 7, cfg)
    sample, idx = O.pillarize_kitti(frame, cfg.grid_spec())
    out = {"cfg": cfg, "graph": graph, "frame": frame, "sample": sample, "idx": idx}
    for key, (label, n_calib) in PLANS.items():
        calib = [pm.make_frame(N_POINTS, 900 + i, cfg, outlier_frac=0.01) for i in range(n_calib)]
        ranges = O.per_sample_ranges(graph, [O.pillarize_kitti(f, cfg.grid_spec())[0] for f in calib])
        stats = pm.calibration.stats_from_ranges(graph, ranges, per_channel_weights=True)
        planned = pm.apply_plan(pm.fold_all_bn(graph), pm.parse_plan_label(label))
        precs = {l.index: l.precision.value for l in planned.weight_layers}
        og = O.folded_graph(planned, precs)
        seen = {}
        ref32 = O.forward(og, sample, stats=stats, observe_fn=lambda l, x: seen.__setitem__(l.index, x))
        with O.accumulate_in(np.float64):
            ref64 = O.forward(og, sample, stats=stats)
        with O.accumulate_in("int"):
            refint = O.forward(og, sample, stats=stats)
        out[key] = {"label": label, "stats": stats, "planned": planned, "precs": precs, "og": og,
                    "inputs": seen, "ref32": ref32, "ref64": ref64, "refint": refint}
    return out


@pytest.mark.parametrize("key", list(PLANS))
def test_end_to_end_headline_config(pm, setup, key):
    cfg, c = setup["cfg"], setup[key]
    eng = pm.PointPillarsEngine(setup["graph"], c["label"], c["stats"], cfg, batch=1,
                                max_points_per_frame=N_POINTS)
    eng.load_points([setup["frame"]])
    eng.run()
    pil = {k: v.cpu().numpy() for k, v in eng.pillars().items()}
    P = int(pil["n_pillars"][0])
    assert P == len(setup["idx"].coords) == MAX_PILLARS  # the cap binds at 120k points
    np.testing.assert_array_equal(pil["coords"][0, :P], setup["idx"].coords)
    np.testing.assert_array_equal(pil["pt_idx"][0, :P], setup["idx"].pt_idx)
    heads = {k: v.cpu().numpy()[0] for k, v in eng.heads_nchw().items()}
    for name, r32, r64, ri in zip(pm.pointpillars.HEADS, c["ref32"], c["ref64"], c["refint"]):
        got = heads[name]
        e_int = rel_l2(got, ri[0])
        e_ref = rel_l2(got, r32[0])
        floor = rel_l2(r32[0], r64[0])
        print(f"{key} {name}: engine-vs-int {e_int:.3e} engine-vs-ref {e_ref:.3e} "
              f"ref-f32-vs-f64 floor {floor:.3e} bar {max(1e-2, 1.1 * floor):.3e}")
        if key == "C2":
            np.testing.assert_array_equal(got, ri[0])  # exact integer execution
        else:
            assert e_int <= 2e-4, (name, e_int)
        assert e_ref <= max(1e-2, 1.1 * floor), (name, e_ref, floor)
    # top-k: the engine's anchor index set == the integer oracle's top-k
    want = O.topk_anchor_order(c["refint"][2][0], cfg.topk)
    got = eng.topk()["idx"][0].cpu().numpy()
    assert set(got.tolist()) == set(want.tolist())
    if key == "C2":
        np.testing.assert_array_equal(got, want)  # identical heads -> identical order


# ----------------------------------------------------------------------------- T1 at full shapes


def _consumers(graph):
    """value name -> consumer weight layers (the DAG rule of pm/model.py:310-367 + inputs)."""
    cons, current, trunk = {}, None, None
    for l in graph.layers:
        if l.inputs:
            srcs = list(l.inputs)
        elif l.is_head:
            trunk = current if trunk is None else trunk
            srcs = [trunk]
        else:
            srcs = [current]
        for s in srcs:
            if s is not None:
                cons.setdefault(s, []).append(l)
        if not l.is_head:
            current = l.name
    # glue values pass their consumers through (maxpool/scatter of the PFN, concat)
    names = {l.name: l for l in graph.layers}

    def weight_consumers(name):
        out = []
        for c in cons.get(name, []):
            out += [c] if c.is_weight_layer else weight_consumers(c.name)
        return out

    return weight_consumers


def _fmt_key(layer, stats):
    p = layer.precision.value
    return ("int8", float(stats[layer.index].act_qp.scale)) if p == "int8" else (p, None)


def _dummy(pm, name, index, cin, fmt):
    """A 1x1 consumer whose only role is to make the producer write `fmt`."""
    w = np.full((16, cin, 1, 1), 0.01, np.float32)
    prec = pm.DType.INT8 if fmt[0] == "int8" else pm.DType(fmt[0])
    # a head: its f32 output is an output of the graph, so every dummy stays live
    return pm.LayerSpec(name=name, kind="conv2d", index=index, weight=w, bias=np.zeros(16, np.float32),
                        conv=pm.ConvParams(), precision=prec, inputs=("L",), is_head=True)


def _run_single(pm, layer, x, stats_l, consumer_fmts, pfn_sample=None):
    """Engine run of `layer` alone on input x with dummy consumers in every format the
    full graph's consumers need.  Returns (f32 output NHWC, {fmt: consumer buffer})."""
    import torch

    from paper_2601_12638_b200 import engine as E

    lay = dataclasses.replace(layer, name="L", index=1, inputs=None)
    cout = lay.weight.shape[0]
    st = {1: stats_l}
    layers = [lay]
    if pfn_sample is not None:
        layers += [pm.LayerSpec(name="mp", kind="maxpool"), pm.LayerSpec(name="sc", kind="scatter",
                                                                         grid=tuple(pfn_sample.grid))]
    src = layers[-1].name
    for j, f in enumerate(consumer_fmts):
        d = _dummy(pm, f"D{j}", 2 + j, cout, f)
        layers.append(dataclasses.replace(d, inputs=(src,)))
        st[2 + j] = O.LayerStats(2 + j, d.name, O._Obs(-1.0, 1.0, 1), O._QP(f[1] or 1.0),
                                 O._PCQP(np.full(16, 0.01 / 127)))
    graph = pm.ModelGraph(layers=tuple(layers))
    stats = O.Stats(layers=st)
    outs = {}
    # (a) production epilogue: the layer's value written only in its consumers' formats
    if consumer_fmts:
        if pfn_sample is not None:
            P, M, F = pfn_sample.features.shape
            grid = E.GridSpec(grid=tuple(pfn_sample.grid), origin=(0.0, 0.0), cell=(1.0, 1.0), max_points=M,
                              max_pillars=None)
            cg = E.CompiledGraph(graph, stats, source="sample", batch=1, grid=grid, pcap=P, n_features=F)
            cg.features[0, :P].copy_(torch.from_numpy(np.ascontiguousarray(pfn_sample.features, np.float32)))
            cg.mask[0, :P].copy_(torch.from_numpy(np.asarray(pfn_sample.point_mask, np.uint8)))
            cg.coords[0, :P].copy_(torch.from_numpy(np.asarray(pfn_sample.coords, np.int64).astype(np.int32)))
            cg.n_pillars.fill_(P)
        else:
            cg = E.CompiledGraph(graph, stats, source="array", in_shape=x.shape)
            cg.input_f32.copy_(torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 3, 1))))
        cg.launch()
        torch.cuda.synchronize()
        v = cg.values[src]
        for f in consumer_fmts:
            t, cs, off = v.bufs[f]
            outs[f] = t[..., off:off + v.shape[3]].cpu().numpy()
    # (b) the layer's f32 output (the final value of a graph without consumers)
    single = pm.ModelGraph(layers=tuple(layers[: 3 if pfn_sample is not None else 1]))
    y = pm.forward(single, pfn_sample if pfn_sample is not None else x, stats=O.Stats(layers={1: stats_l}))
    y = y[0] if isinstance(y, tuple) else y
    return np.ascontiguousarray(np.asarray(y).transpose(0, 2, 3, 1)), outs


@pytest.mark.parametrize("key", list(PLANS))
def test_teacher_forced_every_layer_full_shape(pm, setup, key):
    c = setup[key]
    planned, stats = c["planned"], c["stats"]
    weight_consumers = _consumers(planned)
    og_layers = {l.name: l for l in c["og"].layers}
    report = []
    for layer in planned.weight_layers:
        x = c["inputs"][layer.index]
        value = "middle_encoder.scatter" if layer.index == 1 else layer.name
        fmts = list(dict.fromkeys(_fmt_key(cl, stats) for cl in weight_consumers(value)))
        fmts = [f for f in fmts if f[0] != "fp32"]
        pfn = setup["sample"] if layer.index == 1 else None
        y_e, bufs = _run_single(pm, layer, x, stats[layer.index], fmts, pfn)
        ol = og_layers[layer.name]
        # oracle outputs of the same layer on the same input (NHWC)
        if pfn is not None:
            def ref_of(acc):
                with O.accumulate_in(acc):
                    z = O.run_weight_layer(ol, x, stats)
                return O.scatter_pillars(O.max_over_points(z, pfn.point_mask), pfn.coords, pfn.grid)
        else:
            def ref_of(acc):
                with O.accumulate_in(acc):
                    return O.run_weight_layer(ol, x, stats)
        nhwc = (lambda a: a.transpose(0, 2, 3, 1))
        y32, y64, yint = (np.ascontiguousarray(nhwc(ref_of(a))) for a in (np.float32, np.float64, "int"))
        prec = c["precs"][layer.index]
        row = {"layer": layer.index, "prec": prec, "rel_vs_ref32": rel_l2(y_e, y32)}
        assert row["rel_vs_ref32"] <= 1e-5, row
        if prec == "int8":
            np.testing.assert_array_equal(y_e, yint, err_msg=f"layer {layer.index} f32 output vs integer oracle")
        elif prec == "fp16":
            row["rel_vs_ref64"] = rel_l2(y_e, y64)
            assert row["rel_vs_ref64"] <= 1e-5, row
        for f, buf in bufs.items():
            if f[0] == "int8":
                want = O.quantize(yint if prec == "int8" else y64, f[1]).astype(np.int8)
                flips = float(np.mean(buf != want))
                row[f"flip_int8_vs_oracle@{f[1]:.3g}"] = flips
                row["flip_int8_vs_ref32"] = float(np.mean(O.quantize(y32, f[1]).astype(np.int8) != buf))
                if prec == "int8":
                    assert flips == 0.0, row  # exact codes of the exact output
                    np.testing.assert_array_equal(buf, O.quantize(y_e, f[1]).astype(np.int8))
                else:
                    assert flips <= 1e-4, row
            else:  # fp16 consumer: binary16 of the same output
                got16 = buf.astype(np.float32)
                np.testing.assert_array_equal(got16, O.fp16_roundtrip(y_e))
                if prec == "int8":
                    np.testing.assert_array_equal(got16, O.fp16_roundtrip(yint))
        report.append(row)
    for row in report:
        print(key, row)
