"""Golden vectors for the GPU QAT path (pm/qat.py), produced by the REFERENCE package.

Run in the build container, where the read-only reference exists:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_qat_golden.py
It imports the real pillarmix (never copied) and stores, for the toy detector of
tests/golden/toy.mpq (folded) and a small conv chain:
  * one example's forward-with-tape outputs, detection_loss and backward gradients
    under the FP32 / INT8 (per-tensor and per-channel) / "FP16: 1,12,3" plans;
  * train_qat results (final weights, per-epoch losses) for two configurations
    (plain SGD; momentum + gradient-norm clip over two epochs);
  * ste_fake_quant_backward on values sitting exactly on the clip bounds;
  * mse_loss training of a head-less conv / upsample chain.
Calibration stats are written with the reference's save_stats (calib-stats.json).
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
from pillarmix import qat as QT  # noqa: E402
from pillarmix.calibration import run_calibration, save_stats  # noqa: E402
from pillarmix.detector import DetectorConfig, build_toy_detector, make_train_examples  # noqa: E402
from pillarmix.model import (LayerSpec, ModelGraph, PrecisionPlan, apply_plan, fold_all_bn, forward,  # noqa: E402
                             parse_plan_label, save_model)
from pillarmix.quant import DType  # noqa: E402
from pillarmix.scenes import DatasetConfig, generate_dataset  # noqa: E402
from pillarmix.tensor_ops import ConvParams  # noqa: E402

OUT = Path(__file__).resolve().parent
PLANS = {"FP32": PrecisionPlan(), "INT8": PrecisionPlan(default=DType.INT8),
         "FP16_1_12_3": parse_plan_label("FP16: 1,12,3")}


def toy_qat(data: dict):
    cfg = DetectorConfig()
    graph = fold_all_bn(build_toy_detector(cfg, seed=0))  # == tests/golden/toy.mpq, folded
    scenes = generate_dataset(DatasetConfig(size=6), seed=11)
    examples = make_train_examples(scenes, cfg)
    for i, ex in enumerate(examples):
        s = ex.sample
        data[f"ex{i}_feat"], data[f"ex{i}_mask"], data[f"ex{i}_coords"] = s.features, s.point_mask, s.coords
        data[f"ex{i}_cls_t"], data[f"ex{i}_reg_t"] = ex.cls_target, ex.reg_target
        data[f"ex{i}_pos"], data[f"ex{i}_ign"] = ex.pos_mask, ex.ignore_mask
    stats = run_calibration(graph, [e.sample for e in examples[:4]], seed=0)
    stats_pc = run_calibration(graph, [e.sample for e in examples[:4]], seed=0, per_channel_weights=True)
    save_stats(stats, OUT / "qat_stats.json")
    save_stats(stats_pc, OUT / "qat_stats_pc.json")
    tcfg = QT.TrainConfig()
    cases = dict(PLANS)
    cases["INT8PC"] = PrecisionPlan(default=DType.INT8)
    for pname, plan in cases.items():
        st = stats_pc if pname == "INT8PC" else stats
        g = apply_plan(graph, plan)
        for i in (0, 3):
            tape = []
            outs = forward(g, examples[i].sample, stats=st, tape=tape)
            loss, (dc, dr) = QT.detection_loss(outs, examples[i], tcfg)
            grads = QT.backward(tape, (dc, dr))
            key = f"{pname}_{i}"
            data[f"fw_{key}_cls"], data[f"fw_{key}_reg"] = outs
            data[f"loss_{key}"] = np.float64(loss)
            data[f"dcls_{key}"], data[f"dreg_{key}"] = dc, dr
            for idx, (dw, db) in grads.items():
                data[f"gw_{key}_{idx}"], data[f"gb_{key}_{idx}"] = dw, db
    runs = {
        "sgd_INT8": (PrecisionPlan(default=DType.INT8), stats,
                     QT.TrainConfig(learning_rate=2e-3, epochs=1, batch_size=2, seed=0)),
        "mom_MIX": (parse_plan_label("FP16: 1,12,3"), stats_pc,
                    QT.TrainConfig(learning_rate=5e-3, epochs=2, batch_size=4, seed=3, momentum=0.9,
                                   max_grad_norm=2.0)),
    }
    for rname, (plan, st, tc) in runs.items():
        tuned, hist = QT.train_qat(graph, plan, st, examples, tc)
        data[f"hist_{rname}"] = np.array([h["loss"] for h in hist])
        for l in tuned.weight_layers:
            data[f"tw_{rname}_{l.index}"], data[f"tb_{rname}_{l.index}"] = l.weight, l.bias


def ste_vectors(data: dict):
    rng = np.random.default_rng(7)
    s = 0.0371
    qp = Q.QuantParams(scale=s)
    lo, hi = qp.q_min * s, qp.q_max * s
    x = np.concatenate([rng.uniform(-6, 6, 3000),
                        [lo, hi, np.nextafter(np.float32(lo), np.float32(0)), np.nextafter(np.float32(hi), np.float32(9)),
                         np.float32(lo), np.float32(hi), 0.0, -0.0]]).astype(np.float32)
    up = rng.normal(size=x.shape).astype(np.float32)
    data["ste_x"], data["ste_up"], data["ste_scale"] = x, up, np.float64(s)
    data["ste_out"] = QT.ste_fake_quant_backward(x, qp, up)
    w = rng.normal(size=(6, 4, 3, 3)).astype(np.float32)
    pc = Q.weight_quant_params(w * 0.5, per_channel=True)
    w[0, 0, 0, 0] = np.float32(pc.scales[0] * 127)  # on the bound (as f32)
    w[1, 0, 0, 0] = np.float32(pc.scales[1] * -128)
    upw = rng.normal(size=w.shape).astype(np.float32)
    data["stepc_w"], data["stepc_up"], data["stepc_scales"] = w, upw, pc.scales
    data["stepc_out"] = QT.ste_fake_quant_backward(w, pc, upw)


def chain_qat(data: dict):
    """A head-less conv chain trained with mse_loss (pm/qat.py:119-125)."""
    rng = np.random.default_rng(21)

    def conv(name, idx, cout, cin, k, stride, pad, relu):
        return LayerSpec(name=name, kind="conv2d", index=idx,
                         weight=(rng.normal(size=(cout, cin, k, k)) / np.sqrt(cin * k * k)).astype(np.float32),
                         bias=rng.normal(scale=0.1, size=cout).astype(np.float32), relu=relu,
                         conv=ConvParams(stride=(stride, stride), padding=(pad, pad)))

    layers = (conv("c1", 1, 8, 3, 3, 2, 1, True), conv("c2", 2, 8, 8, 3, 1, 1, True),
              LayerSpec(name="up", kind="upsample2x"), conv("c3", 3, 2, 8, 1, 1, 0, False))
    graph = ModelGraph(layers=layers, meta={})
    save_model(graph, OUT / "qat_chain")
    xs = [rng.normal(size=(1, 3, 10, 12)).astype(np.float32) for _ in range(4)]
    tg = [rng.normal(size=(1, 2, 10, 12)).astype(np.float32) for _ in range(4)]
    for i, (x, t) in enumerate(zip(xs, tg)):
        data[f"chain_x{i}"], data[f"chain_t{i}"] = x, t
    stats = run_calibration(graph, xs, seed=0)
    save_stats(stats, OUT / "qat_chain_stats.json")
    exs = [QT.TrainExample(sample=x, target=t) for x, t in zip(xs, tg)]
    for pname, plan in (("FP32", PrecisionPlan()), ("INT8", PrecisionPlan(default=DType.INT8))):
        tape = []
        out = forward(apply_plan(graph, plan), xs[0], stats=stats, tape=tape)
        loss, grad = QT.mse_loss(out, exs[0], QT.TrainConfig())
        grads = QT.backward(tape, grad)
        data[f"chain_out_{pname}"], data[f"chain_loss_{pname}"] = out, np.float64(loss)
        for idx, (dw, db) in grads.items():
            data[f"chain_gw_{pname}_{idx}"], data[f"chain_gb_{pname}_{idx}"] = dw, db
        tuned, hist = QT.train_qat(graph, plan, stats, exs,
                                   QT.TrainConfig(learning_rate=1e-2, epochs=2, batch_size=2, seed=5),
                                   loss_fn=QT.mse_loss)
        data[f"chain_hist_{pname}"] = np.array([h["loss"] for h in hist])
        for l in tuned.weight_layers:
            data[f"chain_tw_{pname}_{l.index}"], data[f"chain_tb_{pname}_{l.index}"] = l.weight, l.bias


if __name__ == "__main__":
    out: dict = {}
    toy_qat(out)
    ste_vectors(out)
    chain_qat(out)
    np.savez_compressed(OUT / "ref_qat.npz", **out)
    (OUT / "ref_qat_meta.json").write_text(json.dumps({
        "examples": 6, "grad_examples": [0, 3], "plans": list(PLANS) + ["INT8PC"],
        "runs": {"sgd_INT8": {"plan": "INT8", "stats": "qat_stats.json", "learning_rate": 2e-3, "epochs": 1,
                              "batch_size": 2, "seed": 0},
                 "mom_MIX": {"plan": "FP16: 1,12,3", "stats": "qat_stats_pc.json", "learning_rate": 5e-3,
                             "epochs": 2, "batch_size": 4, "seed": 3, "momentum": 0.9, "max_grad_norm": 2.0}},
        "chain": {"learning_rate": 1e-2, "epochs": 2, "batch_size": 2, "seed": 5}}, indent=2) + "\n")
    for p in sorted(OUT.iterdir()):
        if "qat" in p.name:
            print(p.name, p.stat().st_size)
