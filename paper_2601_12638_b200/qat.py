"""Quantization-aware fine-tuning on the GPU (pm/qat.py:1-306).

Same contract as the reference: the forward runs every layer under its plan
precision (INT8: fake-quantised input and weight with the frozen calibrated
scales; FP16: binary16 round trips; FP32: pass-through) and records a tape; the
backward treats each fake-quant node as a clipped straight-through estimator
and the FP16 round trip as identity; plain SGD (optional momentum and gradient
norm clip) updates weights and biases, scales stay frozen.

B200 side: every tensor of the tape lives in HBM and every op is a libpmx
kernel (csrc/train.cu: pre-activation conv / deconv / linear forward, data and
weight gradients, STE masks, max-pool / scatter / upsample / concat adjoints,
the f64 detection and MSE losses, gradient norm, SGD); activations are NHWC,
weights keep the model's [Cout, Cin, kh, kw] layout.  Reductions have a fixed
order, so a run is bit-reproducible; against the reference (numpy f32 BLAS)
results differ only by f32 summation order.

Host side mirrors pm/qat.py: ``TrainConfig``, ``TrainExample``,
``ste_fake_quant_backward``, ``detection_loss``, ``mse_loss``, ``backward``,
``train_qat``; ``model.forward(..., tape=list)`` records this module's
``TapeEntry`` records.  The graph may also be the KITTI extension (deconv2d,
concat).
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass
from typing import Any, Callable, Sequence

import numpy as np

from . import _native as N
from .model import ModelGraph, PrecisionPlan, apply_plan
from .quant import (
    DType,
    PerChannelQuantParams,
    QuantParams,
    fake_quant,
    fake_quant_per_channel,
    fp16_roundtrip,
)

__all__ = [
    "GradState",
    "TapeEntry",
    "TrainConfig",
    "TrainExample",
    "backward",
    "detection_loss",
    "forward_tape",
    "mse_loss",
    "ste_fake_quant_backward",
    "train_qat",
]


@dataclass(frozen=True)
class TrainConfig:
    """pm/qat.py:34-52 (same defaults and validation)."""

    learning_rate: float = 2e-4
    epochs: int = 1
    batch_size: int = 4
    seed: int = 0
    cls_weight: float = 1.0
    reg_weight: float = 5.0
    pos_weight: float = 4.0
    momentum: float = 0.0
    max_grad_norm: float = 0.0

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise ValueError(f"learning_rate must be positive, got {self.learning_rate}")
        if self.epochs < 1:
            raise ValueError(f"epochs must be >= 1, got {self.epochs}")
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError(f"momentum must lie in [0, 1), got {self.momentum}")


@dataclass
class TrainExample:
    """Forward input plus whichever targets the loss consumes (pm/qat.py:55-64)."""

    sample: Any
    cls_target: np.ndarray | None = None
    reg_target: np.ndarray | None = None
    pos_mask: np.ndarray | None = None
    ignore_mask: np.ndarray | None = None
    target: np.ndarray | None = None


GradState = dict  # index -> (dW, db): device f32 tensors in the model's weight layout


# ---------------------------------------------------------------------------
# device activations


@dataclass
class Act:
    """A device activation: ``t`` f32, channel-minor.  ``shape`` is the reference's
    logical shape -- (N, C, H, W) for maps (stored NHWC) or the row shape
    (..., C) of linear / max-pool tensors (stored as is)."""

    t: Any
    shape: tuple
    nchw: bool

    @property
    def c(self) -> int:
        return self.shape[1] if self.nchw else self.shape[-1]

    @property
    def rows(self) -> int:  # pixels (maps) or rows, times c = numel
        return self.t.numel() // max(self.c, 1)

    def numpy(self) -> np.ndarray:
        a = self.t.detach().cpu().numpy()
        if self.nchw:
            n, c, h, w = self.shape
            return np.ascontiguousarray(a.reshape(n, h, w, c).transpose(0, 3, 1, 2))
        return a.reshape(self.shape)

    def like(self, t) -> "Act":
        return Act(t, self.shape, self.nchw)


def _act_from_host(a) -> Act:
    import torch

    a = np.asarray(a, dtype=np.float32)
    if a.ndim == 4:
        t = torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 3, 1))).cuda()
        return Act(t, a.shape, True)
    return Act(torch.from_numpy(np.ascontiguousarray(a)).cuda(), a.shape, False)


def _as_act(x, shape: tuple, nchw: bool) -> Act:
    """A gradient given by the caller (an Act, a CUDA tensor in this engine's layout, or
    an array in the reference's layout) -> an Act of the given logical shape."""
    import torch

    if isinstance(x, Act):
        return x
    numel = int(np.prod(shape))
    if isinstance(x, torch.Tensor) and x.is_cuda and x.numel() == numel and (
            not nchw or tuple(x.shape) != tuple(shape)):
        return Act(x.to(torch.float32).contiguous().reshape(-1), tuple(shape), nchw)
    a = np.asarray(x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else x, dtype=np.float32)
    if a.shape != tuple(shape):
        raise ValueError(f"gradient shape {a.shape} != output shape {tuple(shape)}")
    if nchw:
        return _act_from_host(a)
    return Act(torch.from_numpy(np.ascontiguousarray(a)).cuda(), tuple(shape), False)


def _lib():
    return N.require_cuda()


def _s():
    return N.stream_ptr()


def _empty_like(t):
    import torch

    return torch.empty_like(t)


# ---------------------------------------------------------------------------
# tape


@dataclass
class TapeEntry:
    """Per-layer forward record (pm/model.py:238-249) with device tensors, plus the
    graph wiring (value names) and the kernel geometry of this engine."""

    layer: Any
    x_in: Any = None        # Act: input before any precision transform
    x_used: Any = None      # Act: input fed to the kernel
    w_used: Any = None      # device f32 weight after the precision transform
    pre_act: Any = None     # Act: kernel output + bias, before ReLU
    act_qp: QuantParams | None = None
    weight_qp: QuantParams | PerChannelQuantParams | None = None
    argmax: Any = None      # device int32 [P, C] max-pool winners
    sample: Any = None      # device int32 coords [P, 2] (scatter)
    src: tuple = ()         # value names consumed
    out: str = ""           # value name produced
    desc: Any = None        # N.ConvDesc of weight layers
    weight: Any = None      # the layer's current f32 weight on the device (STE mask)
    out_shape: tuple = ()   # logical output shape
    out_nchw: bool = False  # output stored NHWC with an (N, C, H, W) logical shape


def _desc_for(layer, x: Act) -> tuple[Any, tuple, bool]:
    """(ConvDesc, logical output shape, nchw) for a weight layer on input x."""
    w = layer.weight
    if layer.kind == "linear":
        if x.nchw:
            raise ValueError(f"linear layer {layer.name!r} expects a row tensor, got a 4D map")
        din = x.shape[-1]
        if din != w.shape[1]:
            raise ValueError(f"linear input features {din} != weight in-features {w.shape[1]}")
        rows = x.rows
        d = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.PMX_F32, batch=rows, in_h=1, in_w=1, in_c=din, in_c_stride=din,
                       in_c_offset=0, out_c=w.shape[0], k_h=1, k_w=1, stride_h=1, stride_w=1, pad_h=0, pad_w=0,
                       out_h=1, out_w=1, relu=0)
        return d, tuple(x.shape[:-1]) + (w.shape[0],), False
    if not x.nchw:
        raise ValueError(f"{layer.kind} expects 4D input/weight, got {tuple(x.shape)} and {w.shape}")
    n, c, h, wd = x.shape
    f, cw, kh, kw = w.shape
    if c != cw:
        raise ValueError(f"{layer.kind} input channels {c} != weight channels {cw}")
    sh, sw = layer.conv.stride
    if layer.kind == "deconv2d":
        if (kh, kw) != (sh, sw):
            raise ValueError("deconv2d supports kernel == stride only")
        oh, ow, ph, pw = h * sh, wd * sw, 0, 0
        kind = N.PMX_DECONV2D
    else:
        ph, pw = layer.conv.padding
        oh, ow = layer.conv.out_size((h, wd), (kh, kw))
        kind = N.PMX_CONV2D
    d = N.ConvDesc(kind=kind, in_dtype=N.PMX_F32, batch=n, in_h=h, in_w=wd, in_c=c, in_c_stride=c, in_c_offset=0,
                   out_c=f, k_h=kh, k_w=kw, stride_h=sh, stride_w=sw, pad_h=ph, pad_w=pw, out_h=oh, out_w=ow, relu=0)
    return d, (n, f, oh, ow), True


def _layer_quant(layer, stats):
    """pm/model.py:261-267 (same error)."""
    if stats is None or layer.index not in stats:
        raise RuntimeError(
            f"layer {layer.index} ({layer.name!r}) is tagged int8 but calibration "
            "stats supply no quant params for it"
        )
    entry = stats[layer.index]
    return entry.act_qp, entry.weight_qp


def _weight_forward(layer, x: Act, stats, weights, tape):
    """pm/model.py:270-307 on the device: precision transform, conv, ReLU, tape."""
    import torch

    lib = _lib()
    if layer.bn is not None:
        raise ValueError(f"layer {layer.name!r} still carries batch norm; fold before training")
    w, b = weights[layer.index]
    act_qp = weight_qp = None
    prec = layer.precision
    if prec is DType.INT8:
        act_qp, weight_qp = _layer_quant(layer, stats)
        x_used = x.like(fake_quant(x.t, act_qp))
        if isinstance(weight_qp, PerChannelQuantParams):
            w_used = fake_quant_per_channel(w, weight_qp)
        else:
            w_used = fake_quant(w, weight_qp)
    elif prec is DType.FP16:
        x_used = x.like(fp16_roundtrip(x.t))
        w_used = fp16_roundtrip(w)
    else:
        x_used, w_used = x, w
    desc, oshape, nchw = _desc_for(layer, x)
    numel = int(np.prod(oshape))
    pre = torch.empty(numel, dtype=torch.float32, device="cuda")
    N.check(lib.pmx_train_conv_fwd(desc, x_used.t.data_ptr(), w_used.data_ptr(), b.data_ptr(), pre.data_ptr(), _s()),
            layer.name)
    pre_act = Act(pre, oshape, nchw)
    out = pre_act
    if layer.relu:
        r = torch.empty_like(pre)
        N.check(lib.pmx_train_relu(pre.data_ptr(), numel, r.data_ptr(), _s()), layer.name)
        out = Act(r, oshape, nchw)
    if tape is not None:
        tape.append(TapeEntry(layer=layer, x_in=x, x_used=x_used, w_used=w_used, pre_act=pre_act, act_qp=act_qp,
                              weight_qp=weight_qp, desc=desc, weight=w, out_shape=oshape))
    return out


def _device_weights(graph: ModelGraph) -> dict:
    import torch

    out = {}
    for l in graph.weight_layers:
        out[l.index] = (torch.from_numpy(np.ascontiguousarray(l.weight, np.float32)).cuda(),
                        torch.from_numpy(np.ascontiguousarray(l.bias, np.float32)).cuda())
    return out


def forward_tape(graph: ModelGraph, x, stats=None, tape: list | None = None, weights: dict | None = None):
    """pm/model.py:310-367 on the device, recording ``tape`` (TapeEntry per layer).

    Returns the head outputs (or the final output) as device ``Act`` records; use
    ``Act.numpy()`` for the reference's NCHW / row arrays.  ``weights`` maps a layer
    index to its device (weight, bias) (default: uploaded from the graph)."""
    import torch

    lib = _lib()
    if weights is None:
        weights = _device_weights(graph)
    sample = x if hasattr(x, "point_mask") else None
    coords = None
    if sample is not None:
        current = _act_from_host(np.asarray(sample.features, np.float32))
        mask = torch.from_numpy(np.ascontiguousarray(sample.point_mask, np.uint8)).cuda()
        coords_np = np.asarray(sample.coords, np.int64).reshape(-1, 2)
    else:
        current = _act_from_host(np.asarray(x, dtype=np.float32))
    values = {"__input__": current}
    cur_name = "__input__"
    trunk = None
    heads = []
    for layer in graph.layers:
        if layer.inputs:
            src_names = tuple(layer.inputs)
        elif layer.is_head:
            trunk = cur_name if trunk is None else trunk
            src_names = (trunk,)
        else:
            src_names = (cur_name,)
        src = values[src_names[0]]
        n0 = len(tape) if tape is not None else 0
        if layer.is_weight_layer:
            out = _weight_forward(layer, src, stats, weights, tape)
        elif layer.kind == "maxpool":
            if sample is None:
                raise ValueError(f"maxpool layer {layer.name!r} needs a PillarSample input")
            P, M, C = src.shape
            if P and not np.asarray(sample.point_mask).any(axis=1).all():
                raise ValueError("pillar with no real points cannot be max-pooled")
            o = torch.empty(P * C, dtype=torch.float32, device="cuda")
            arg = torch.empty(P * C, dtype=torch.int32, device="cuda")
            N.check(lib.pmx_train_maxpool(src.t.data_ptr(), mask.data_ptr(), P, M, C, o.data_ptr(), arg.data_ptr(),
                                          _s()), layer.name)
            out = Act(o, (P, C), False)
            if tape is not None:
                tape.append(TapeEntry(layer=layer, x_in=src, argmax=arg, out_shape=(P, C)))
        elif layer.kind == "scatter":
            if sample is None:
                raise ValueError(f"scatter layer {layer.name!r} needs a PillarSample input")
            if layer.grid is not None and tuple(layer.grid) != tuple(sample.grid):
                raise ValueError(f"scatter grid {layer.grid} does not match sample grid {sample.grid}")
            H, W = sample.grid
            P, C = src.shape
            bad = (coords_np[:, 0] < 0) | (coords_np[:, 0] >= H) | (coords_np[:, 1] < 0) | (coords_np[:, 1] >= W)
            if bad.any():
                i = int(np.argmax(bad))
                raise ValueError(f"pillar coord {tuple(coords_np[i])} outside grid {tuple(sample.grid)}")
            if len(np.unique(coords_np[:, 0] * W + coords_np[:, 1])) != P:
                raise ValueError("duplicate pillar coords")
            if coords is None:
                coords = torch.from_numpy(coords_np.astype(np.int32)).cuda()
            o = torch.zeros(H * W * C, dtype=torch.float32, device="cuda")
            N.check(lib.pmx_train_scatter(src.t.data_ptr(), coords.data_ptr(), P, C, W, o.data_ptr(), _s()),
                    layer.name)
            out = Act(o, (1, C, H, W), True)
            if tape is not None:
                tape.append(TapeEntry(layer=layer, x_in=src, sample=coords, out_shape=out.shape))
        elif layer.kind == "upsample2x":
            n, c, h, w = src.shape
            o = torch.empty(n * 4 * h * w * c, dtype=torch.float32, device="cuda")
            N.check(lib.pmx_upsample2x(src.t.data_ptr(), N.PMX_F32, n, h, w, c, o.data_ptr(), _s()), layer.name)
            out = Act(o, (n, c, 2 * h, 2 * w), True)
            if tape is not None:
                tape.append(TapeEntry(layer=layer, x_in=src, out_shape=out.shape))
        elif layer.kind == "concat":
            parts = [values[n_] for n_ in src_names]
            n, _, h, w = parts[0].shape
            ctot = sum(p.shape[1] for p in parts)
            o = torch.empty(n * h * w * ctot, dtype=torch.float32, device="cuda")
            off = 0
            for p in parts:
                if p.shape[0] != n or p.shape[2:] != (h, w):
                    raise ValueError(f"concat {layer.name!r}: input extents differ")
                c = p.shape[1]
                N.check(lib.pmx_train_copy_channels(p.t.data_ptr(), n * h * w, c, c, 0, o.data_ptr(), ctot, off,
                                                    _s()), layer.name)
                off += c
            out = Act(o, (n, ctot, h, w), True)
            if tape is not None:
                tape.append(TapeEntry(layer=layer, out_shape=out.shape))
        else:
            raise ValueError(f"layer {layer.name!r}: kind {layer.kind!r} has no training path")
        if tape is not None and len(tape) > n0:
            tape[-1].src = src_names
            tape[-1].out = layer.name
            tape[-1].out_nchw = out.nchw
        values[layer.name] = out
        if layer.is_head:
            heads.append(out)
        else:
            cur_name = layer.name
    if heads:
        return tuple(heads)
    return values[cur_name]


# ---------------------------------------------------------------------------
# losses


def _outputs_host(outputs):
    if isinstance(outputs, tuple):
        return tuple(o.numpy() if isinstance(o, Act) else np.asarray(o) for o in outputs)
    return outputs.numpy() if isinstance(outputs, Act) else np.asarray(outputs)


def _nhwc64(a, hw_shape):
    """[C, H, W] -> contiguous f64 [H, W, C] on the device."""
    import torch

    a = np.asarray(a, dtype=np.float64).reshape((-1,) + tuple(hw_shape))
    return torch.from_numpy(np.ascontiguousarray(a.transpose(1, 2, 0))).cuda()


def _ws():
    import torch

    return torch.empty(_lib().pmx_train_reduce_workspace() // 8, dtype=torch.float64, device="cuda")


def detection_loss(outputs, example: TrainExample, cfg: TrainConfig):
    """Weighted BCE on the class map plus MSE on box offsets at positive cells, both
    normalised by the number of positive cells (pm/qat.py:92-116), on the device.

    ``outputs`` = (cls_map, reg_map): device ``Act`` records (the training loop) or
    the reference's NCHW arrays; the gradients come back in the same form."""
    import torch

    lib = _lib()
    host = not isinstance(outputs[0], Act)
    cls = outputs[0] if not host else _act_from_host(outputs[0])
    reg = outputs[1] if not host else _act_from_host(outputs[1])
    _, ncls, H, W = cls.shape
    nreg = reg.shape[1]
    pos = np.asarray(example.pos_mask)
    n_pos = max(1, int(pos.sum()))
    t = _nhwc64(example.cls_target, (H, W))
    rt = _nhwc64(example.reg_target, (H, W))
    pos_d = torch.from_numpy(np.ascontiguousarray(pos.reshape(H, W), np.uint8)).cuda()
    ign = None
    if example.ignore_mask is not None:
        ign = torch.from_numpy(np.ascontiguousarray(np.asarray(example.ignore_mask).reshape(H, W), np.uint8)).cuda()
    d_cls = torch.empty_like(cls.t)
    d_reg = torch.empty_like(reg.t)
    sums = torch.empty(2, dtype=torch.float64, device="cuda")
    N.check(lib.pmx_train_detection_loss(cls.t.data_ptr(), t.data_ptr(), N.ptr(ign), pos_d.data_ptr(), reg.t.data_ptr(),
                                         rt.data_ptr(), H * W, ncls, nreg, float(n_pos), float(cfg.cls_weight),
                                         float(cfg.reg_weight), float(cfg.pos_weight), d_cls.data_ptr(),
                                         d_reg.data_ptr(), sums.data_ptr(), _ws().data_ptr(), _s()), "detection_loss")
    s = sums.cpu().numpy()
    cls_loss = float(s[0] / n_pos)
    reg_loss = float(s[1] / (4.0 * n_pos))
    loss = cfg.cls_weight * cls_loss + cfg.reg_weight * reg_loss
    dc, dr = cls.like(d_cls), reg.like(d_reg)
    if host:
        return loss, (dc.numpy(), dr.numpy())
    return loss, (dc, dr)


def mse_loss(outputs, example: TrainExample, cfg: TrainConfig):
    """Mean squared error against ``example.target`` (pm/qat.py:119-125), on the device."""
    import torch

    lib = _lib()
    out = outputs[0] if isinstance(outputs, tuple) else outputs
    host = not isinstance(out, Act)
    o = _act_from_host(out) if host else out
    tgt = np.asarray(example.target, dtype=np.float64)
    if tgt.shape != tuple(o.shape):
        tgt = np.broadcast_to(tgt, o.shape)
    if o.nchw:
        tgt = tgt.transpose(0, 2, 3, 1)
    td = torch.from_numpy(np.ascontiguousarray(tgt)).cuda()
    g = torch.empty_like(o.t)
    s = torch.empty(1, dtype=torch.float64, device="cuda")
    N.check(lib.pmx_train_mse_loss(o.t.data_ptr(), td.data_ptr(), o.t.numel(), g.data_ptr(), s.data_ptr(),
                                   _ws().data_ptr(), _s()), "mse_loss")
    loss = float(s.cpu().numpy()[0] / o.t.numel())
    ga = o.like(g)
    return loss, (ga.numpy() if host else ga)


# ---------------------------------------------------------------------------
# backward


def ste_fake_quant_backward(x, qp, upstream):
    """Clipped STE: pass ``upstream`` through where x sits inside the clip range
    (pm/qat.py:79-85).  numpy in -> numpy out; CUDA tensors stay on the device."""
    import torch

    lib = _lib()
    as_np = not isinstance(x, torch.Tensor)
    xs = np.shape(x) if as_np else tuple(x.shape)
    us = np.shape(upstream) if not isinstance(upstream, torch.Tensor) else tuple(upstream.shape)
    if xs != us:
        raise ValueError(f"STE shape mismatch: x {xs} vs upstream {us}")
    xd = torch.as_tensor(np.ascontiguousarray(x, np.float32) if as_np else x, dtype=torch.float32).contiguous().cuda()
    ud = torch.as_tensor(np.ascontiguousarray(upstream, np.float32) if not isinstance(upstream, torch.Tensor)
                         else upstream, dtype=torch.float32).contiguous().cuda()
    out = torch.empty_like(ud)
    _ste(lib, xd, qp, ud, out)
    return out.cpu().numpy() if as_np else out


def _ste(lib, x, qp, up, out, rows: int | None = None):
    """out = up * in_range(x, qp) on the device; per-channel rows = leading extent."""
    import torch

    n = x.numel()
    if isinstance(qp, PerChannelQuantParams):
        r = rows if rows is not None else x.shape[0]
        sc = torch.from_numpy(np.ascontiguousarray(qp.scales, np.float64)).cuda()
        N.check(lib.pmx_train_ste_rows(x.data_ptr(), r, n // max(r, 1), sc.data_ptr(), int(qp.q_min), int(qp.q_max),
                                       up.data_ptr(), out.data_ptr(), _s()), "ste")
    else:
        N.check(lib.pmx_train_ste(x.data_ptr(), n, float(qp.scale), int(qp.q_min), int(qp.q_max), up.data_ptr(),
                                  out.data_ptr(), _s()), "ste")


def _weight_backward(lib, e: TapeEntry, dout: Act, grads: dict, need_dx: bool):
    """pm/qat.py:155-172: ReLU mask, data + weight gradients, STE for INT8 layers."""
    import torch

    layer = e.layer
    if layer.bn is not None:
        raise ValueError(f"layer {layer.name!r} still carries batch norm; fold before training")
    d = dout.t
    if layer.relu:
        m = torch.empty_like(d)
        N.check(lib.pmx_train_relu_bwd(d.data_ptr(), e.pre_act.t.data_ptr(), d.numel(), m.data_ptr(), _s()),
                layer.name)
        d = m
    dw = torch.empty_like(e.w_used)
    db = torch.empty(layer.bias.shape[0], dtype=torch.float32, device="cuda")
    N.check(lib.pmx_train_conv_wgrad(e.desc, d.data_ptr(), e.x_used.t.data_ptr(), dw.data_ptr(), db.data_ptr(), _s()),
            layer.name)
    dx = None
    if need_dx:
        dxu = torch.empty_like(e.x_used.t)
        N.check(lib.pmx_train_conv_dgrad(e.desc, d.data_ptr(), e.w_used.data_ptr(), dxu.data_ptr(), _s()), layer.name)
        dx = dxu
    if e.act_qp is not None:  # int8: clipped STE through both fake-quant nodes
        if dx is not None:
            m = torch.empty_like(dx)
            _ste(lib, e.x_in.t, e.act_qp, dx, m)
            dx = m
        m = torch.empty_like(dw)
        _ste(lib, e.weight, e.weight_qp, dw, m, rows=layer.weight.shape[0])
        dw = m
    old = grads.get(layer.index)
    if old is None:
        grads[layer.index] = (dw, db)
    else:
        aw, ab = torch.empty_like(dw), torch.empty_like(db)
        N.check(lib.pmx_train_add(old[0].data_ptr(), dw.data_ptr(), dw.numel(), aw.data_ptr(), _s()), "grad acc")
        N.check(lib.pmx_train_add(old[1].data_ptr(), db.data_ptr(), db.numel(), ab.data_ptr(), _s()), "grad acc")
        grads[layer.index] = (aw, ab)
    return None if dx is None else e.x_in.like(dx)


def _accumulate(lib, dgrads: dict, name: str, g: Act):
    """Gradient of a value consumed more than once: summed in processing order
    (the reference's d_trunk + d_in over the heads, pm/qat.py:199-210)."""
    import torch

    old = dgrads.get(name)
    if old is None:
        dgrads[name] = g
        return
    s = torch.empty_like(old.t)
    N.check(lib.pmx_train_add(old.t.data_ptr(), g.t.data_ptr(), s.numel(), s.data_ptr(), _s()), "grad acc")
    dgrads[name] = old.like(s)


def backward(tape: list, d_outputs) -> GradState:
    """Weight / bias gradients from the output gradients over a tape (pm/qat.py:199-222).

    ``d_outputs``: one gradient per head in head order (or one for a head-less graph),
    device ``Act`` records, CUDA tensors or the reference's arrays.  Returns
    {index: (dW, db)} as device tensors."""
    import torch

    lib = _lib()
    grads: GradState = {}
    if not tape:
        return grads
    dgrads: dict = {}
    head_entries = [e for e in tape if e.layer.is_head]
    if head_entries:
        douts = list(d_outputs) if isinstance(d_outputs, (tuple, list)) else [d_outputs]
        if len(douts) != len(head_entries):
            raise ValueError(f"{len(douts) - len(head_entries)} output gradients left over after heads"
                             if len(douts) > len(head_entries) else "missing output gradients")
        for e, d in zip(head_entries, douts):
            dgrads[e.out] = _as_act(d, e.out_shape, e.out_nchw)
    else:
        d = d_outputs if not isinstance(d_outputs, (tuple, list)) else d_outputs[0]
        last = tape[-1]
        dgrads[last.out] = _as_act(d, last.out_shape, last.out_nchw)
    consumed = {n for e in tape for n in e.src}
    for e in reversed(tape):
        g = dgrads.pop(e.out, None)
        if g is None:  # output feeds nothing the loss sees
            continue
        src = e.src[0] if e.src else "__input__"
        need_dx = src != "__input__" and src in consumed
        kind = e.layer.kind
        if e.layer.is_weight_layer:
            dx = _weight_backward(lib, e, g, grads, need_dx)
            if dx is not None:
                _accumulate(lib, dgrads, src, dx)
        elif kind == "maxpool":
            P, M, C = e.x_in.shape
            dx = torch.empty(P * M * C, dtype=torch.float32, device="cuda")
            N.check(lib.pmx_train_maxpool_bwd(g.t.data_ptr(), e.argmax.data_ptr(), P, M, C, dx.data_ptr(), _s()),
                    e.layer.name)
            if need_dx:
                _accumulate(lib, dgrads, src, e.x_in.like(dx))
        elif kind == "scatter":
            P, C = e.x_in.shape
            W = e.out_shape[3]
            dx = torch.empty(P * C, dtype=torch.float32, device="cuda")
            N.check(lib.pmx_train_scatter_bwd(g.t.data_ptr(), e.sample.data_ptr(), P, C, W, dx.data_ptr(), _s()),
                    e.layer.name)
            if need_dx:
                _accumulate(lib, dgrads, src, e.x_in.like(dx))
        elif kind == "upsample2x":
            n, c, h, w = e.x_in.shape
            dx = torch.empty(n * h * w * c, dtype=torch.float32, device="cuda")
            N.check(lib.pmx_train_upsample2x_bwd(g.t.data_ptr(), n, h, w, c, dx.data_ptr(), _s()), e.layer.name)
            if need_dx:
                _accumulate(lib, dgrads, src, e.x_in.like(dx))
        elif kind == "concat":
            n, ctot, h, w = e.out_shape
            off = 0
            for name in e.src:
                part_shape = None
                for t in tape:
                    if t.out == name:
                        part_shape = t.out_shape
                c = part_shape[1]
                dx = torch.empty(n * h * w * c, dtype=torch.float32, device="cuda")
                N.check(lib.pmx_train_copy_channels(g.t.data_ptr(), n * h * w, c, ctot, off, dx.data_ptr(), c, 0, _s()),
                        e.layer.name)
                _accumulate(lib, dgrads, name, Act(dx, part_shape, True))
                off += c
    return grads


# ---------------------------------------------------------------------------
# training loop


def _trainable_copy(graph: ModelGraph) -> ModelGraph:
    layers = [dataclasses.replace(l, weight=l.weight.copy(), bias=l.bias.copy()) if l.is_weight_layer else l
              for l in graph.layers]
    return ModelGraph(layers=tuple(layers), meta=graph.meta)


def _sync_host(g: ModelGraph, weights: dict):
    """Device weights -> the graph's arrays, in place (the evaluator sees the tuned graph)."""
    for l in g.weight_layers:
        w, b = weights[l.index]
        l.weight[...] = w.cpu().numpy().reshape(l.weight.shape)
        l.bias[...] = b.cpu().numpy().reshape(l.bias.shape)


def train_qat(
    graph: ModelGraph,
    plan: PrecisionPlan,
    stats,
    data: Sequence[TrainExample],
    cfg: TrainConfig,
    loss_fn: Callable = detection_loss,
    evaluator: Callable | None = None,
) -> tuple[ModelGraph, list[dict]]:
    """Fine-tune weights under the plan's precision, scales frozen (pm/qat.py:239-306).

    Returns the tuned graph and the per-epoch history (mean train loss, evaluator
    score or None).  A ``loss_fn`` other than this module's losses receives the
    reference's host arrays and may return host gradients."""
    import torch

    lib = _lib()
    if any(l.bn is not None for l in graph.layers):
        raise ValueError("fold batch norm before training")
    if not data:
        raise ValueError("training data is empty")
    g = _trainable_copy(apply_plan(graph, plan))
    weights = _device_weights(g)
    velocity: dict = {}
    history: list[dict] = []
    native_loss = loss_fn in (detection_loss, mse_loss)
    ws = _ws()
    tot = torch.empty(1, dtype=torch.float64, device="cuda")
    for epoch in range(cfg.epochs):
        rng = np.random.default_rng((cfg.seed, epoch))
        order = rng.permutation(len(data))
        epoch_losses = []
        for b_start in range(0, len(order), cfg.batch_size):
            batch = order[b_start: b_start + cfg.batch_size]
            acc: dict = {}
            batch_loss = 0.0
            for si in batch:
                example = data[int(si)]
                tape: list = []
                outputs = forward_tape(g, example.sample, stats=stats, tape=tape, weights=weights)
                if native_loss:
                    loss, d_outputs = loss_fn(outputs, example, cfg)
                else:
                    loss, d_outputs = loss_fn(_outputs_host(outputs), example, cfg)
                if not math.isfinite(loss):
                    raise RuntimeError(
                        f"non-finite train loss at epoch {epoch}, "
                        f"batch {b_start // cfg.batch_size}, sample {int(si)}"
                    )
                batch_loss += loss
                for index, (dw, db) in backward(tape, d_outputs).items():
                    old = acc.get(index)
                    if old is None:
                        acc[index] = (dw, db)
                    else:
                        aw, ab = torch.empty_like(dw), torch.empty_like(db)
                        N.check(lib.pmx_train_add(old[0].data_ptr(), dw.data_ptr(), dw.numel(), aw.data_ptr(), _s()))
                        N.check(lib.pmx_train_add(old[1].data_ptr(), db.data_ptr(), db.numel(), ab.data_ptr(), _s()))
                        acc[index] = (aw, ab)
            inv = np.float32(1.0 / len(batch))
            if cfg.max_grad_norm > 0.0:
                total_sq = 0.0
                for dw, db in acc.values():
                    for t in (dw, db):
                        N.check(lib.pmx_train_sumsq(t.data_ptr(), t.numel(), float(inv), tot.data_ptr(),
                                                    ws.data_ptr(), _s()), "grad norm")
                        total_sq += float(tot.cpu().numpy()[0])
                total = math.sqrt(total_sq)
                if total > cfg.max_grad_norm:
                    inv = np.float32(inv * cfg.max_grad_norm / total)
            lr = np.float32(cfg.learning_rate)
            mu = np.float32(cfg.momentum)
            for index, (dw, db) in acc.items():
                w, b = weights[index]
                if cfg.momentum > 0.0 and index not in velocity:
                    velocity[index] = (torch.zeros_like(w), torch.zeros_like(b))
                vw, vb = velocity.get(index, (None, None))
                for t, gr, v in ((w, dw, vw), (b, db, vb)):
                    N.check(lib.pmx_train_sgd(t.data_ptr(), gr.data_ptr(), t.numel(), float(inv), float(lr), float(mu),
                                              N.ptr(v), _s()), "sgd")
            epoch_losses.append(batch_loss / len(batch))
        _sync_host(g, weights)
        score = float(evaluator(g, plan, stats)) if evaluator is not None else None
        history.append({"epoch": epoch, "loss": float(np.mean(epoch_losses)), "score": score})
    torch.cuda.synchronize()
    return g, history
