"""QAT on the GPU (pm/qat.py) against the reference.

Golden vectors come from the real pillarmix (tests/golden/make_qat_golden.py): the
toy detector's forward-with-tape outputs, detection loss and backward gradients under
four plans, two full train_qat runs (plain SGD; momentum + gradient clip over two
epochs), the clipped-STE mask on values sitting exactly on the clip bounds, and a
head-less conv chain trained with mse_loss.  The element-wise pieces (STE, loss
gradients) are bit-exact; everything downstream of an f32 matrix product differs from
numpy's BLAS only by summation order, measured as relative L2 error against a bar
written in each test.  The KITTI extension (deconv2d, concat, three heads) has no
reference QAT counterpart: its gradients are checked against torch f64 autograd of
the same forward.
"""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


@pytest.fixture(scope="module")
def ref():
    return dict(np.load(GOLDEN / "ref_qat.npz"))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n > 0 else d


def _examples(pm, ref):
    from paper_2601_12638_b200.qat import TrainExample

    out = []
    for i in range(6):
        s = pm.PillarSample(features=ref[f"ex{i}_feat"], point_mask=ref[f"ex{i}_mask"], coords=ref[f"ex{i}_coords"],
                            grid=(16, 16))
        out.append(TrainExample(sample=s, cls_target=ref[f"ex{i}_cls_t"], reg_target=ref[f"ex{i}_reg_t"],
                                pos_mask=ref[f"ex{i}_pos"], ignore_mask=ref[f"ex{i}_ign"]))
    return out


def _plan(pm, name):
    return {"FP32": pm.PrecisionPlan(), "INT8": pm.PrecisionPlan(default=pm.DType.INT8),
            "INT8PC": pm.PrecisionPlan(default=pm.DType.INT8),
            "FP16_1_12_3": pm.parse_plan_label("FP16: 1,12,3")}[name]


def test_ste_golden_bit_exact(pm, ref):
    from paper_2601_12638_b200.qat import ste_fake_quant_backward

    got = ste_fake_quant_backward(ref["ste_x"], pm.QuantParams(scale=float(ref["ste_scale"])), ref["ste_up"])
    np.testing.assert_array_equal(got, ref["ste_out"])
    got = ste_fake_quant_backward(ref["stepc_w"], pm.PerChannelQuantParams(scales=ref["stepc_scales"]),
                                  ref["stepc_up"])
    np.testing.assert_array_equal(got, ref["stepc_out"])
    with pytest.raises(ValueError, match="STE shape mismatch"):
        ste_fake_quant_backward(ref["ste_x"][:5], pm.QuantParams(scale=0.1), ref["ste_up"][:4])


# Bars: FP32 / FP16 forwards differ from the reference's BLAS by f32 reassociation only
# (<= 1e-5 on the head maps); INT8 forwards may flip a near-tie activation code, whose
# effect is one quantisation step at one element (<= 1e-3).  Loss gradients are
# element-wise f64 -> f32 on those maps (same bars); weight / bias gradients sum over
# every pixel (measured <= 1e-6 on B200; bars 2e-5 FP32/FP16, 1e-4 INT8).
@pytest.mark.parametrize("plan", ["FP32", "INT8", "INT8PC", "FP16_1_12_3"])
@pytest.mark.parametrize("i", [0, 3])
def test_toy_forward_loss_backward(pm, ref, plan, i):
    from paper_2601_12638_b200 import qat

    graph = pm.fold_all_bn(pm.load_model(GOLDEN / "toy"))
    stats = pm.load_stats(GOLDEN / ("qat_stats_pc.json" if plan == "INT8PC" else "qat_stats.json"))
    g = pm.apply_plan(graph, _plan(pm, plan))
    ex = _examples(pm, ref)[i]
    tape = []
    cls, reg = pm.forward(g, ex.sample, stats=stats, tape=tape)
    key = f"{plan}_{i}"
    fw_bar = 1e-3 if plan.startswith("INT8") else 1e-5
    assert rel_l2(cls, ref[f"fw_{key}_cls"]) <= fw_bar
    assert rel_l2(reg, ref[f"fw_{key}_reg"]) <= fw_bar
    loss, (dc, dr) = qat.detection_loss((cls, reg), ex, qat.TrainConfig())
    assert abs(loss - float(ref[f"loss_{key}"])) <= fw_bar * abs(float(ref[f"loss_{key}"]))
    assert rel_l2(dc, ref[f"dcls_{key}"]) <= fw_bar and rel_l2(dr, ref[f"dreg_{key}"]) <= fw_bar
    # the loss kernel alone is exact: the reference's own maps in, its gradients out
    _, (dc0, dr0) = qat.detection_loss((ref[f"fw_{key}_cls"], ref[f"fw_{key}_reg"]), ex, qat.TrainConfig())
    assert np.array_equal(dc0, ref[f"dcls_{key}"]) or rel_l2(dc0, ref[f"dcls_{key}"]) <= 1e-7
    assert np.array_equal(dr0, ref[f"dreg_{key}"])
    grads = qat.backward(tape, (dc, dr))
    assert sorted(grads) == sorted(int(k.split("_")[-1]) for k in ref if k.startswith(f"gw_{key}_"))
    g_bar = 1e-4 if plan.startswith("INT8") else 2e-5
    worst = 0.0
    for idx, (dw, db) in grads.items():
        ew = rel_l2(dw.cpu().numpy().reshape(ref[f"gw_{key}_{idx}"].shape), ref[f"gw_{key}_{idx}"])
        eb = rel_l2(db.cpu().numpy(), ref[f"gb_{key}_{idx}"])
        worst = max(worst, ew, eb)
    print(f"{key}: worst grad rel-L2 {worst:.2e}")
    assert worst <= g_bar


def _stats_for(pm, name):
    return pm.load_stats(GOLDEN / name)


# Two optimiser steps per epoch compound the reassociation differences; the bar is
# on the weight UPDATE (tuned - initial), relative to the reference's update.
@pytest.mark.parametrize("run", ["sgd_INT8", "mom_MIX"])
def test_train_qat_matches_reference(pm, ref, run):
    from paper_2601_12638_b200 import qat

    meta = json.loads((GOLDEN / "ref_qat_meta.json").read_text())["runs"][run]
    graph = pm.fold_all_bn(pm.load_model(GOLDEN / "toy"))
    plan = pm.parse_plan_label(meta["plan"])
    stats = _stats_for(pm, meta["stats"])
    cfg = qat.TrainConfig(learning_rate=meta["learning_rate"], epochs=meta["epochs"], batch_size=meta["batch_size"],
                          seed=meta["seed"], momentum=meta.get("momentum", 0.0),
                          max_grad_norm=meta.get("max_grad_norm", 0.0))
    tuned, hist = qat.train_qat(graph, plan, stats, _examples(pm, ref), cfg)
    np.testing.assert_allclose([h["loss"] for h in hist], ref[f"hist_{run}"], rtol=2e-3)
    assert all(h["score"] is None for h in hist)
    base = {l.index: l for l in pm.apply_plan(graph, plan).weight_layers}
    worst = 0.0
    for l in tuned.weight_layers:
        for got, want, init in ((l.weight, ref[f"tw_{run}_{l.index}"], base[l.index].weight),
                                (l.bias, ref[f"tb_{run}_{l.index}"], base[l.index].bias)):
            upd_ref = want.astype(np.float64) - init
            if np.linalg.norm(upd_ref) == 0:
                np.testing.assert_array_equal(got, want)
                continue
            worst = max(worst, rel_l2(got.astype(np.float64) - init, upd_ref))
    print(f"{run}: worst update rel-L2 {worst:.2e}")
    assert worst <= 1e-3  # measured 1.3e-5
    # the input graph is untouched; a second run is bit-identical (fixed-order reductions)
    assert np.array_equal(graph.layers[0].weight, pm.fold_all_bn(pm.load_model(GOLDEN / "toy")).layers[0].weight)
    tuned2, _ = qat.train_qat(graph, plan, stats, _examples(pm, ref), cfg)
    for a, b in zip(tuned.weight_layers, tuned2.weight_layers):
        assert np.array_equal(a.weight, b.weight) and np.array_equal(a.bias, b.bias)


def test_chain_mse_training(pm, ref):
    from paper_2601_12638_b200 import qat

    graph = pm.load_model(GOLDEN / "qat_chain")
    stats = pm.load_stats(GOLDEN / "qat_chain_stats.json")
    xs = [ref[f"chain_x{i}"] for i in range(4)]
    exs = [qat.TrainExample(sample=x, target=ref[f"chain_t{i}"]) for i, x in enumerate(xs)]
    meta = json.loads((GOLDEN / "ref_qat_meta.json").read_text())["chain"]
    for pname in ("FP32", "INT8"):
        plan = _plan(pm, pname)
        g = pm.apply_plan(graph, plan)
        tape = []
        out = pm.forward(g, xs[0], stats=stats, tape=tape)
        bar = 1e-3 if pname == "INT8" else 1e-5
        assert rel_l2(out, ref[f"chain_out_{pname}"]) <= bar
        loss, grad = qat.mse_loss(out, exs[0], qat.TrainConfig())
        assert abs(loss - float(ref[f"chain_loss_{pname}"])) <= bar * float(ref[f"chain_loss_{pname}"])
        grads = qat.backward(tape, grad)
        for idx, (dw, db) in grads.items():
            assert rel_l2(dw.cpu().numpy().reshape(ref[f"chain_gw_{pname}_{idx}"].shape),
                          ref[f"chain_gw_{pname}_{idx}"]) <= 10 * bar
            assert rel_l2(db.cpu().numpy(), ref[f"chain_gb_{pname}_{idx}"]) <= 10 * bar
        tuned, hist = qat.train_qat(graph, plan, stats, exs,
                                    qat.TrainConfig(learning_rate=meta["learning_rate"], epochs=meta["epochs"],
                                                    batch_size=meta["batch_size"], seed=meta["seed"]),
                                    loss_fn=qat.mse_loss)
        np.testing.assert_allclose([h["loss"] for h in hist], ref[f"chain_hist_{pname}"], rtol=10 * bar)
        for l in tuned.weight_layers:
            init = graph.layer_by_index(l.index)
            assert rel_l2(l.weight.astype(np.float64) - init.weight,
                          ref[f"chain_tw_{pname}_{l.index}"].astype(np.float64) - init.weight) <= 1e-2
            assert rel_l2(l.bias.astype(np.float64) - init.bias,
                          ref[f"chain_tb_{pname}_{l.index}"].astype(np.float64) - init.bias) <= 1e-2


def test_custom_loss_and_errors(pm, ref):
    """A user loss gets the reference's host arrays; non-finite losses, unfolded BN and
    empty data raise the reference's errors."""
    from paper_2601_12638_b200 import qat

    graph = pm.fold_all_bn(pm.load_model(GOLDEN / "toy"))
    stats = pm.load_stats(GOLDEN / "qat_stats.json")
    exs = _examples(pm, ref)[:2]
    seen = []

    def my_loss(outputs, example, cfg):
        seen.append(tuple(o.shape for o in outputs))
        return qat.detection_loss(outputs, example, cfg)

    _, hist = qat.train_qat(graph, pm.PrecisionPlan(), stats, exs, qat.TrainConfig(batch_size=2), loss_fn=my_loss)
    assert seen and seen[0] == (ref["fw_FP32_0_cls"].shape, ref["fw_FP32_0_reg"].shape)
    assert np.isfinite(hist[0]["loss"])

    def bad_loss(outputs, example, cfg):
        return float("nan"), tuple(np.zeros_like(o) for o in outputs)

    with pytest.raises(RuntimeError, match="non-finite train loss at epoch 0, batch 0, sample"):
        qat.train_qat(graph, pm.PrecisionPlan(), stats, exs, qat.TrainConfig(), loss_fn=bad_loss)
    with pytest.raises(ValueError, match="fold batch norm before training"):
        qat.train_qat(pm.load_model(GOLDEN / "toy"), pm.PrecisionPlan(), stats, exs, qat.TrainConfig())
    with pytest.raises(ValueError, match="training data is empty"):
        qat.train_qat(graph, pm.PrecisionPlan(), stats, [], qat.TrainConfig())
    with pytest.raises(RuntimeError, match="tagged int8 but calibration"):
        pm.forward(pm.apply_plan(graph, pm.PrecisionPlan(default=pm.DType.INT8)), exs[0].sample, stats=None, tape=[])


def _torch_reference_grads(graph, sample, r_heads):
    """f64 autograd of the same forward (FP32 plan, BN folded) -- the KITTI extension's
    oracle for the backward: loss = sum_h <out_h, R_h>."""
    import torch
    import torch.nn.functional as F

    P = sample.features.shape[0]
    params = {}
    for l in graph.weight_layers:
        params[l.index] = (torch.tensor(l.weight, dtype=torch.float64, requires_grad=True),
                           torch.tensor(l.bias, dtype=torch.float64, requires_grad=True))
    mask = torch.tensor(np.asarray(sample.point_mask, bool))
    coords = torch.tensor(np.asarray(sample.coords, np.int64))
    vals = {"__input__": torch.tensor(sample.features, dtype=torch.float64)}
    cur, trunk, heads = "__input__", None, []
    for l in graph.layers:
        if l.inputs:
            src = list(l.inputs)
        elif l.is_head:
            trunk = cur if trunk is None else trunk
            src = [trunk]
        else:
            src = [cur]
        x = vals[src[0]]
        if l.kind == "linear":
            w, b = params[l.index]
            y = x @ w.T + b
        elif l.kind == "conv2d":
            w, b = params[l.index]
            y = F.conv2d(x, w, b, stride=l.conv.stride, padding=l.conv.padding)
        elif l.kind == "deconv2d":
            w, b = params[l.index]
            y = F.conv_transpose2d(x, w.transpose(0, 1), b, stride=l.conv.stride)
        elif l.kind == "maxpool":
            y = torch.where(mask[:, :, None], x, torch.tensor(-np.inf, dtype=torch.float64)).max(dim=1).values
        elif l.kind == "scatter":
            H, W = sample.grid
            flat = torch.zeros(x.shape[1], H * W, dtype=torch.float64)
            flat[:, coords[:, 0] * W + coords[:, 1]] = x.T
            y = flat.reshape(1, x.shape[1], H, W)
        elif l.kind == "concat":
            y = torch.cat([vals[n] for n in src], dim=1)
        elif l.kind == "upsample2x":
            y = x.repeat_interleave(2, dim=2).repeat_interleave(2, dim=3)
        else:
            raise AssertionError(l.kind)
        if l.is_weight_layer and l.relu:
            y = torch.relu(y)
        vals[l.name] = y
        if l.is_head:
            heads.append(y)
        else:
            cur = l.name
    loss = sum((h * torch.tensor(r, dtype=torch.float64)).sum() for h, r in zip(heads, r_heads))
    loss.backward()
    return {i: (w.grad.numpy(), b.grad.numpy()) for i, (w, b) in params.items()}, [h.detach().numpy() for h in heads]


def test_kitti_extension_grads_vs_autograd(pm):
    """Deconvs, the concat and three heads (no reference QAT counterpart): the GPU tape
    backward against torch f64 autograd of the same FP32 forward (<= 1e-4 rel-L2)."""
    from oracle import pillars_oracle as O
    from paper_2601_12638_b200 import qat

    cfg = pm.PointPillarsConfig.small(grid=(32, 24), max_pillars=400)
    graph = pm.fold_all_bn(pm.build_pointpillars(cfg, seed=4))
    sample, _ = O.pillarize_kitti(pm.make_frame(1500, 8, cfg), cfg.grid_spec())
    tape = []
    outs = pm.forward(graph, sample, tape=tape)
    rng = np.random.default_rng(2)
    rs = [rng.normal(size=o.shape).astype(np.float32) for o in outs]
    want, heads = _torch_reference_grads(graph, sample, rs)
    for o, h in zip(outs, heads):
        assert rel_l2(o, h) <= 1e-5
    grads = qat.backward(tape, tuple(rs))
    assert sorted(grads) == sorted(want)
    for idx, (dw, db) in grads.items():
        assert rel_l2(dw.cpu().numpy().reshape(want[idx][0].shape), want[idx][0]) <= 1e-4, idx
        assert rel_l2(db.cpu().numpy(), want[idx][1]) <= 1e-4, idx
