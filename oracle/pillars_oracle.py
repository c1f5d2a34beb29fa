"""CPU oracle for the pillarize -> forward -> decode hot path (TEST INFRASTRUCTURE ONLY).

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it.  The product package
(``paper_2601_12638_b200``) never imports anything under ``oracle/``.

It restates, in numpy, the reference package ``pillarmix``
(``/root/reference/pkg/src/pillarmix``, abbreviated ``pm/`` below) and
extends it to the KITTI-shaped PointPillars the north star names (SURVEY.md
§8(c) "What must be restated").  Every function cites the reference line it
follows.  Pinning: ``tests/golden/make_golden.py`` imports the real reference
in the build container and writes fixtures; ``tests/test_oracle_golden.py``
checks this module against them bit-exactly (quant math, tensor ops, chain
forward on the reference toy detector, 5-feature pillarize, toy decode).  The
KITTI extensions (9 features, pillar cap, deconv, concat DAG, anchor top-k)
have no reference counterpart: they reduce to the pinned pieces (the cap is
the identity when it does not bind; deconv is ``linear`` + reshape; the DAG
executor is the chain executor when ``inputs`` is absent) and are otherwise
"parity unpinned" as DESIGN.md records.

Duck typing: graph / layer / stats objects may come from either the reference
package or the product package; only attribute names are used.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

Q_MIN = -128
Q_MAX = 127
FP16_MAX = 65504.0


# ---------------------------------------------------------------------------
# quant math: pm/quant.py


def compute_scale(x_min: float, x_max: float) -> float:
    """pm/quant.py:82-95 -- symmetric scale max(|min|,|max|)/127, degenerate -> 1.0."""
    if not (math.isfinite(x_min) and math.isfinite(x_max)):
        raise ValueError(f"non-finite calibration range ({x_min}, {x_max})")
    if x_min > x_max:
        raise ValueError(f"calibration range has min {x_min} > max {x_max}")
    max_abs = max(abs(x_min), abs(x_max))
    if max_abs == 0.0:
        return 1.0
    return max_abs / Q_MAX


def quantize(x, scale: float) -> np.ndarray:
    """pm/quant.py:98-103 -- clip(rint(f64(x) / scale)) as int32 (f64 divide)."""
    xq = np.clip(np.rint(np.asarray(x, dtype=np.float64) / scale), Q_MIN, Q_MAX)
    return xq.astype(np.int32)


def dequantize(codes, scale: float) -> np.ndarray:
    """pm/quant.py:106-111."""
    return np.asarray(codes, dtype=np.float64) * scale


def fake_quant(t, scale: float) -> np.ndarray:
    """pm/quant.py:114-116 -- f32(f64(code) * scale)."""
    return dequantize(quantize(t, scale), scale).astype(np.float32)


def weight_scales(weight: np.ndarray, per_channel: bool):
    """pm/quant.py:119-133 -- per-tensor (range includes 0) or per-axis-0 scales."""
    w = np.asarray(weight, dtype=np.float64)
    if not np.all(np.isfinite(w)):
        raise ValueError("weight tensor contains non-finite values")
    if not per_channel:
        return compute_scale(float(w.min(initial=0.0)), float(w.max(initial=0.0)))
    flat = w.reshape(w.shape[0], -1)
    max_abs = np.abs(flat).max(axis=1)
    return np.where(max_abs == 0.0, 1.0, max_abs / Q_MAX)


def weight_codes_per_channel(weight: np.ndarray, scales: np.ndarray) -> np.ndarray:
    """Integer codes of pm/quant.py:136-141 (before the dequantizing multiply)."""
    w = np.asarray(weight, dtype=np.float64)
    s = np.asarray(scales, dtype=np.float64).reshape((-1,) + (1,) * (w.ndim - 1))
    return np.clip(np.rint(w / s), Q_MIN, Q_MAX).astype(np.int32)


def fake_quant_per_channel(weight: np.ndarray, scales: np.ndarray) -> np.ndarray:
    """pm/quant.py:136-141."""
    w = np.asarray(weight, dtype=np.float64)
    s = np.asarray(scales, dtype=np.float64).reshape((-1,) + (1,) * (w.ndim - 1))
    codes = np.clip(np.rint(w / s), Q_MIN, Q_MAX)
    return (codes * s).astype(np.float32)


def fp16_roundtrip(t) -> np.ndarray:
    """pm/quant.py:144-147 -- clip to +-65504 then RNE binary16 and back."""
    clipped = np.clip(np.asarray(t, dtype=np.float32), -FP16_MAX, FP16_MAX)
    return clipped.astype(np.float16).astype(np.float32)


def minmax(t) -> tuple[float, float]:
    """pm/quant.py:179-188 / pm/calibration.py:116-118 -- exact (min, max); empty -> (0, 0)."""
    t = np.asarray(t)
    if t.size == 0:
        return 0.0, 0.0
    return float(t.min()), float(t.max())


# ---------------------------------------------------------------------------
# tensor ops: pm/tensor_ops.py (f32 NCHW, f32 accumulate)


# Accumulation dtype of the dense kernels.  float32 is the reference (numpy sgemm);
# float64 gives the re-association noise floor SURVEY §8(d) T2 asks to report.
_ACC = {"dtype": np.float32}


class accumulate_in:
    """Context manager: run linear/conv2d/deconv2d products in another dtype, round to f32."""

    def __init__(self, dtype):
        self.dtype = dtype

    def __enter__(self):
        self.prev = _ACC["dtype"]
        _ACC["dtype"] = self.dtype

    def __exit__(self, *exc):
        _ACC["dtype"] = self.prev


def _mm(a, b):
    dt = _ACC["dtype"]
    if dt is np.float32:
        return a @ b
    if isinstance(dt, str):  # "int" probe: non-INT8 layers accumulate in f64
        dt = np.float64
    return (a.astype(dt) @ b.astype(dt)).astype(np.float32)


def linear(x, weight, bias):
    """pm/tensor_ops.py:80-91."""
    x = np.asarray(x, dtype=np.float32)
    return _mm(x, weight.T) + bias


def out_size(in_hw, k_hw, stride, padding):
    """pm/tensor_ops.py:47-57."""
    out = []
    for size, k, s, p in zip(in_hw, k_hw, stride, padding):
        out.append((size + 2 * p - k) // s + 1)
    return out[0], out[1]


def im2col(x, k_hw, stride, padding):
    """pm/tensor_ops.py:94-106 -- K order (c, kh, kw)."""
    kh, kw = k_hw
    ph, pw = padding
    sh, sw = stride
    n, c, h, w = x.shape
    ho, wo = out_size((h, w), (kh, kw), stride, padding)
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    windows = sliding_window_view(xp, (kh, kw), axis=(2, 3))[:, :, ::sh, ::sw]
    windows = windows[:, :, :ho, :wo]
    return np.ascontiguousarray(windows.transpose(0, 2, 3, 1, 4, 5)).reshape(n * ho * wo, c * kh * kw)


def conv2d(x, weight, bias, stride=(1, 1), padding=(0, 0)):
    """pm/tensor_ops.py:109-131 -- im2col + sgemm."""
    x = np.asarray(x, dtype=np.float32)
    n, c, h, w = x.shape
    f, cw, kh, kw = weight.shape
    if c != cw:
        raise ValueError(f"conv2d input channels {c} != weight channels {cw}")
    ho, wo = out_size((h, w), (kh, kw), stride, padding)
    cols = im2col(x, (kh, kw), stride, padding)
    out = _mm(cols, weight.reshape(f, -1).T) + bias
    return np.ascontiguousarray(out.reshape(n, ho, wo, f).transpose(0, 3, 1, 2))


def deconv2d(x, weight, bias, stride):
    """KITTI extension: ConvTranspose2d with kernel == stride.

    Restated through ``linear`` (pm/tensor_ops.py:80-91) + a pixel shuffle.
    weight is stored [Cout, Cin, k, k] so that axis 0 is the output channel
    (per-channel quant axis, pm/quant.py:119-141):
      out[n, co, s*i+dy, s*j+dx] = sum_ci x[n, ci, i, j] * W[co, ci, dy, dx] + b[co]
    """
    x = np.asarray(x, dtype=np.float32)
    n, cin, h, w = x.shape
    cout, cw, kh, kw = weight.shape
    if cin != cw:
        raise ValueError(f"deconv2d input channels {cin} != weight channels {cw}")
    sh, sw = stride
    if (kh, kw) != (sh, sw):
        raise ValueError("deconv2d supports kernel == stride only")
    rows = np.ascontiguousarray(x.transpose(0, 2, 3, 1)).reshape(n * h * w, cin)
    wl = np.ascontiguousarray(weight.transpose(0, 2, 3, 1)).reshape(cout * kh * kw, cin)
    out = linear(rows, wl, np.repeat(np.asarray(bias, np.float32), kh * kw))
    out = out.reshape(n, h, w, cout, kh, kw).transpose(0, 3, 1, 4, 2, 5)
    return np.ascontiguousarray(out.reshape(n, cout, h * kh, w * kw))


def relu(x):
    """pm/tensor_ops.py:134-135."""
    return np.maximum(x, np.float32(0.0))


def scatter_pillars(features, coords, grid):
    """pm/tensor_ops.py:138-160."""
    h, w = grid
    features = np.asarray(features, dtype=np.float32)
    coords = np.asarray(coords, dtype=np.int64).reshape(-1, 2)
    p, c = features.shape
    out = np.zeros((1, c, h, w), dtype=np.float32)
    if p == 0:
        return out
    rows, cols = coords[:, 0], coords[:, 1]
    if ((rows < 0) | (rows >= h) | (cols < 0) | (cols >= w)).any():
        raise ValueError("pillar coord outside grid")
    if len(np.unique(rows * w + cols)) != p:
        raise ValueError("duplicate pillar coords")
    out[0, :, rows, cols] = features
    return out


def max_over_points(features, point_mask):
    """pm/tensor_ops.py:163-173 -- masked max over points."""
    if features.shape[0] == 0:
        return np.zeros((0, features.shape[2]), dtype=np.float32)
    if not point_mask.any(axis=1).all():
        raise ValueError("pillar with no real points cannot be max-pooled")
    masked = np.where(point_mask[:, :, None], features, np.float32(-np.inf))
    return masked.max(axis=1)


def upsample2x(x):
    """pm/tensor_ops.py:176-178."""
    return np.repeat(np.repeat(x, 2, axis=2), 2, axis=3)


# ---------------------------------------------------------------------------
# pillarize: pm/scenes.py:155-193, generalised to an origin offset, 9 features
# and a pillar cap


@dataclass(frozen=True)
class PillarIndex:
    """Integer part of pillarize (the T0 bit-exact tier)."""

    coords: np.ndarray      # [P, 2] int64 (row, col), ascending flat id
    counts: np.ndarray      # [P] int64, kept points (<= M)
    pt_idx: np.ndarray      # [P, M] int64 point indices in scene order, -1 padding
    total_counts: np.ndarray  # [P] int64, all points of the cell (before truncation)


def bin_points(xy: np.ndarray, grid, origin, cell) -> np.ndarray:
    """pm/scenes.py:175-179 -- f32 divide, truncate toward zero, clamp to the grid.

    ``xy`` is [N, 2] float32 (x, y).  ``origin`` = (x_min, y_min), ``cell`` =
    (cell_w, cell_h); all arithmetic in IEEE f32 exactly as NEP 50 evaluates
    ``f32_array / py_float`` in the reference.
    """
    h, w = grid
    x = xy[:, 0].astype(np.float32)
    y = xy[:, 1].astype(np.float32)
    x0, y0 = np.float32(origin[0]), np.float32(origin[1])
    cw, ch = np.float32(cell[0]), np.float32(cell[1])
    with np.errstate(invalid="ignore"):
        fy = np.clip((y - y0) / ch, np.float32(-1.0), np.float32(h))
        fx = np.clip((x - x0) / cw, np.float32(-1.0), np.float32(w))
    rows = np.clip(fy.astype(np.int64), 0, h - 1)
    cols = np.clip(fx.astype(np.int64), 0, w - 1)
    return rows * w + cols


def pillar_index(flat: np.ndarray, grid, max_points: int, max_pillars: int | None) -> PillarIndex:
    """Pillar selection + first-come truncation (pm/scenes.py:180-186).

    Pillars are emitted in ascending flat id (pm/scenes.py:180-183); each keeps
    its first ``max_points`` points in scene order (pm/scenes.py:185).  Cap
    (KITTI extension): when more than ``max_pillars`` cells
    are occupied, keep the ``max_pillars`` cells whose first point has the
    smallest scene index; the reference has no cap, and this rule is the
    identity whenever the cap does not bind.
    """
    h, w = grid
    n = flat.shape[0]
    if n == 0:
        return PillarIndex(
            coords=np.zeros((0, 2), np.int64),
            counts=np.zeros((0,), np.int64),
            pt_idx=np.full((0, max_points), -1, np.int64),
            total_counts=np.zeros((0,), np.int64),
        )
    cells, first_idx, cell_counts = np.unique(flat, return_index=True, return_counts=True)
    if max_pillars is not None and len(cells) > max_pillars:
        keep = np.sort(np.argsort(first_idx, kind="stable")[:max_pillars])
        cells, cell_counts = cells[keep], cell_counts[keep]
    p = len(cells)
    order = np.argsort(flat, kind="stable")          # scene order within a cell
    sorted_flat = flat[order]
    starts = np.searchsorted(sorted_flat, cells, side="left")
    counts = np.minimum(cell_counts, max_points)
    pt_idx = np.full((p, max_points), -1, np.int64)
    slot = np.arange(max_points)
    take = slot[None, :] < counts[:, None]
    src = starts[:, None] + slot[None, :]
    pt_idx[take] = order[src[take]]
    coords = np.stack([cells // w, cells % w], axis=1).astype(np.int64)
    return PillarIndex(coords=coords, counts=counts.astype(np.int64), pt_idx=pt_idx,
                       total_counts=cell_counts.astype(np.int64))


def _gather_mean(vals: np.ndarray, pt_idx: np.ndarray, counts: np.ndarray) -> np.ndarray:
    """Sequential f32 sum over kept points / f32(k): numpy's ``chunk.mean(axis=0)``
    at pm/scenes.py:187 (checked equal for k <= 300 in the build container)."""
    p, m = pt_idx.shape
    acc = np.zeros((p,) + vals.shape[1:], np.float32)
    for s in range(m):
        live = counts > s
        if not live.any():
            break
        acc[live] = (acc[live] + vals[pt_idx[live, s]]).astype(np.float32)
    den = np.maximum(counts, 1).astype(np.float32).reshape((-1,) + (1,) * (vals.ndim - 1))
    return (acc / den).astype(np.float32)


def pillar_features5(points: np.ndarray, idx: PillarIndex) -> tuple[np.ndarray, np.ndarray]:
    """pm/scenes.py:186-192 -- (x, y, i, x-mx, y-my), zero padded, plus mask."""
    p, m = idx.pt_idx.shape
    feats = np.zeros((p, m, 5), np.float32)
    mask = idx.pt_idx >= 0
    if p == 0:
        return feats, mask
    center = _gather_mean(points[:, :2].astype(np.float32), idx.pt_idx, idx.counts)
    g = points[np.where(mask, idx.pt_idx, 0)].astype(np.float32)
    feats[..., 0:3] = g[..., 0:3]
    feats[..., 3:5] = g[..., 0:2] - center[:, None, :]
    feats[~mask] = 0.0
    return feats, mask


def pillar_features9(points: np.ndarray, idx: PillarIndex, origin, cell) -> tuple[np.ndarray, np.ndarray]:
    """KITTI extension: standard PointPillars 9-feature augmentation.

    (x, y, z, r, x-mx, y-my, z-mz, x-xc, y-yc): cluster offsets to the mean of
    the pillar's kept points (same f32 sequential mean as pm/scenes.py:187)
    and xy offsets to the pillar centre xc = f32(col)*cell_w + f32(cell_w/2 +
    x_min) (each op rounded to f32, no fused multiply-add); padding rows are
    zero and masked (pm/scenes.py:189-192).
    """
    p, m = idx.pt_idx.shape
    feats = np.zeros((p, m, 9), np.float32)
    mask = idx.pt_idx >= 0
    if p == 0:
        return feats, mask
    pts = points.astype(np.float32)
    mean = _gather_mean(pts[:, :3], idx.pt_idx, idx.counts)
    g = pts[np.where(mask, idx.pt_idx, 0)]
    cw, ch = np.float32(cell[0]), np.float32(cell[1])
    # offsets from the f32 grid parameters, combined in f64 (pmx_grid carries f32)
    xoff = np.float32(float(np.float32(cell[0])) * 0.5 + float(np.float32(origin[0])))
    yoff = np.float32(float(np.float32(cell[1])) * 0.5 + float(np.float32(origin[1])))
    xc = (idx.coords[:, 1].astype(np.float32) * cw).astype(np.float32) + xoff
    yc = (idx.coords[:, 0].astype(np.float32) * ch).astype(np.float32) + yoff
    feats[..., 0:4] = g[..., 0:4]
    feats[..., 4:7] = g[..., 0:3] - mean[:, None, :]
    feats[..., 7] = g[..., 0] - xc[:, None].astype(np.float32)
    feats[..., 8] = g[..., 1] - yc[:, None].astype(np.float32)
    feats[~mask] = 0.0
    return feats, mask


@dataclass(frozen=True)
class Sample:
    """Duck-typed PillarSample (pm/tensor_ops.py:60-77)."""

    features: np.ndarray
    point_mask: np.ndarray
    coords: np.ndarray
    grid: tuple


def pillarize_ref5(points, grid, max_points_per_pillar, field_size) -> Sample:
    """pm/scenes.py:155-193 exactly (no cap, origin 0, 5 features)."""
    h, w = grid
    pts = np.asarray(points, np.float32)
    cell = (field_size / w, field_size / h)
    flat = bin_points(pts[:, :2], grid, (0.0, 0.0), cell)
    idx = pillar_index(flat, grid, max_points_per_pillar, None)
    feats, mask = pillar_features5(pts, idx)
    return Sample(features=feats, point_mask=mask, coords=idx.coords, grid=tuple(grid))


def pillarize_kitti(points, geom) -> tuple[Sample, PillarIndex]:
    """KITTI-shaped pillarize: ``geom`` has grid, origin, cell, max_points, max_pillars."""
    pts = np.asarray(points, np.float32)
    flat = bin_points(pts[:, :2], geom.grid, geom.origin, geom.cell)
    idx = pillar_index(flat, geom.grid, geom.max_points, geom.max_pillars)
    feats, mask = pillar_features9(pts, idx, geom.origin, geom.cell)
    return Sample(features=feats, point_mask=mask, coords=idx.coords, grid=tuple(geom.grid)), idx


# ---------------------------------------------------------------------------
# model: pm/model.py (fold, precision dispatch, forward), generalised to a DAG


def _prec(layer) -> str:
    p = layer.precision
    return getattr(p, "value", p)


def fold_bn_arrays(weight, bias, gamma, beta, mean, var, eps):
    """pm/model.py:209-225 -- f64 factor rounded to f32, then f32 products."""
    denom_sq = var.astype(np.float64) + eps
    if np.any(denom_sq <= 0):
        raise ValueError("non-positive var + eps")
    factor = (gamma.astype(np.float64) / np.sqrt(denom_sq)).astype(np.float32)
    shape = (-1,) + (1,) * (weight.ndim - 1)
    w = (weight * factor.reshape(shape)).astype(np.float32)
    b = ((bias - mean) * factor + beta).astype(np.float32)
    return w, b


def apply_bn(out, bn, kind):
    """pm/model.py:252-258 (unfolded BN at run time)."""
    factor = (bn.gamma / np.sqrt(bn.var + np.float32(bn.eps))).astype(np.float32)
    if kind in ("conv2d", "deconv2d"):
        shape = (1, -1, 1, 1)
    else:
        shape = (1,) * (out.ndim - 1) + (-1,)
    return (out - bn.mean.reshape(shape)) * factor.reshape(shape) + bn.beta.reshape(shape)


def _stat_scales(layer, stats):
    """pm/model.py:261-268 -- missing stats is a RuntimeError naming the layer."""
    if stats is None or layer.index not in stats:
        raise RuntimeError(
            f"layer {layer.index} ({layer.name!r}) is tagged int8 but calibration "
            "stats supply no quant params for it"
        )
    entry = stats[layer.index]
    act = float(entry.act_qp.scale)
    wqp = entry.weight_qp
    if hasattr(wqp, "scales"):
        return act, np.asarray(wqp.scales, np.float64), True
    return act, float(wqp.scale), False


def transform_input(layer, x, stats):
    """Precision transform of a weight layer's input (pm/model.py:273-285)."""
    p = _prec(layer)
    if p == "int8":
        act, _, _ = _stat_scales(layer, stats)
        return fake_quant(x, act)
    if p == "fp16":
        return fp16_roundtrip(x)
    return np.asarray(x, np.float32)


def transform_weight(layer, stats):
    """Precision transform of a weight layer's weight (pm/model.py:276-282)."""
    p = _prec(layer)
    if p == "int8":
        _, ws, per_channel = _stat_scales(layer, stats)
        if per_channel:
            return fake_quant_per_channel(layer.weight, ws)
        return fake_quant(layer.weight, ws)
    if p == "fp16":
        return fp16_roundtrip(layer.weight)
    return layer.weight


def _int8_layer_integer(layer, x, stats):
    """Integer-execution probe of an INT8 layer (TensorRT-style: exact int32 accumulation of
    codes, then y = f32(acc) * f32(s_x * s_w[c]) + bias in one rounding).  Used only inside
    ``accumulate_in("int")`` to measure how far two valid executions of the same plan drift."""
    act, ws, per_channel = _stat_scales(layer, stats)
    cx = quantize(x, act).astype(np.float64)
    w = np.asarray(layer.weight)
    cw = (weight_codes_per_channel(w, ws) if per_channel else quantize(w, ws)).astype(np.float64)
    cout = w.shape[0]
    alpha = np.asarray(np.float32(act * np.broadcast_to(np.asarray(ws, np.float64), (cout,))), np.float64)
    if layer.kind == "linear":
        acc = cx @ cw.T
        shape = (1,) * (acc.ndim - 1) + (-1,)
    elif layer.kind == "conv2d":
        n, c, h, wd = cx.shape
        ho, wo = out_size((h, wd), w.shape[2:], layer.conv.stride, layer.conv.padding)
        cols = im2col(cx, w.shape[2:], layer.conv.stride, layer.conv.padding)
        acc = (cols @ cw.reshape(cout, -1).T).reshape(n, ho, wo, cout).transpose(0, 3, 1, 2)
        shape = (1, -1, 1, 1)
    else:
        n, cin, h, wd = cx.shape
        kh, kw = w.shape[2:]
        rows = cx.transpose(0, 2, 3, 1).reshape(-1, cin)
        acc = rows @ cw.transpose(0, 2, 3, 1).reshape(cout * kh * kw, cin).T
        acc = acc.reshape(n, h, wd, cout, kh, kw).transpose(0, 3, 1, 4, 2, 5).reshape(n, cout, h * kh, wd * kw)
        shape = (1, -1, 1, 1)
    y = (acc * alpha.reshape(shape) + np.asarray(layer.bias, np.float64).reshape(shape)).astype(np.float32)
    return np.ascontiguousarray(y)


def run_weight_layer(layer, x, stats):
    """pm/model.py:271-307 (kernel dispatch extended with deconv2d)."""
    if isinstance(_ACC["dtype"], str) and _ACC["dtype"] == "int" and _prec(layer) == "int8":
        out = _int8_layer_integer(layer, x, stats)
        if layer.bn is not None:
            out = apply_bn(out, layer.bn, layer.kind)
        return relu(out) if layer.relu else out
    x_used = transform_input(layer, x, stats)
    w_used = transform_weight(layer, stats)
    if layer.kind == "linear":
        out = linear(x_used, w_used, layer.bias)
    elif layer.kind == "conv2d":
        out = conv2d(x_used, w_used, layer.bias, layer.conv.stride, layer.conv.padding)
    elif layer.kind == "deconv2d":
        out = deconv2d(x_used, w_used, layer.bias, layer.conv.stride)
    else:
        raise ValueError(f"unknown weight kind {layer.kind!r}")
    if layer.bn is not None:
        out = apply_bn(out, layer.bn, layer.kind)
    if layer.relu:
        out = relu(out)
    return out


def forward(graph, x, stats=None, observe_fn=None):
    """pm/model.py:310-367, generalised to a DAG.

    A layer without ``inputs`` consumes the previous non-head output (heads
    consume the trunk, pm/model.py:329-331) exactly like the reference chain;
    a layer with ``inputs`` consumes the named layers' outputs (``concat``
    joins them along channels).  ``observe_fn(layer, x)`` sees each weight
    layer's input before its precision transform (pm/model.py:335-336).
    """
    sample = x if hasattr(x, "point_mask") else None
    current = sample.features if sample is not None else np.asarray(x, np.float32)
    outputs: dict[str, np.ndarray] = {}
    heads: list[np.ndarray] = []
    trunk = None
    for layer in graph.layers:
        names = getattr(layer, "inputs", None)
        if names:
            srcs = [outputs[nm] for nm in names]
            source = srcs[0]
        elif layer.is_head:
            trunk = current if trunk is None else trunk
            source = trunk
            srcs = [source]
        else:
            source = current
            srcs = [source]
        kind = layer.kind
        if kind in ("linear", "conv2d", "deconv2d"):
            if observe_fn is not None:
                observe_fn(layer, source)
            out = run_weight_layer(layer, source, stats)
        elif kind == "maxpool":
            out = max_over_points(source, sample.point_mask)
        elif kind == "scatter":
            out = scatter_pillars(source, sample.coords, sample.grid)
        elif kind == "upsample2x":
            out = upsample2x(source)
        elif kind == "concat":
            out = np.concatenate(srcs, axis=1)
        else:
            raise ValueError(f"unknown kind {kind!r}")
        outputs[layer.name] = out
        if layer.is_head:
            heads.append(out)
        else:
            current = out
    if heads:
        return tuple(heads)
    return current


def fold_graph_layers(graph):
    """pm/model.py:228-230 as plain dicts: name -> (weight, bias) folded."""
    out = {}
    for l in graph.layers:
        if l.weight is None:
            continue
        if l.bn is not None:
            w, b = fold_bn_arrays(l.weight, l.bias, l.bn.gamma, l.bn.beta, l.bn.mean, l.bn.var, l.bn.eps)
        else:
            w, b = l.weight, l.bias
        out[l.name] = (w, b)
    return out


# ---------------------------------------------------------------------------
# calibration: pm/calibration.py:106-165 (duck-typed stats records)


@dataclass(frozen=True)
class _QP:
    scale: float


@dataclass(frozen=True)
class _PCQP:
    scales: np.ndarray


@dataclass(frozen=True)
class _Obs:
    running_min: float
    running_max: float
    count: int


@dataclass(frozen=True)
class LayerStats:
    index: int
    name: str
    observer: _Obs
    act_qp: _QP
    weight_qp: object


@dataclass(frozen=True)
class Stats:
    layers: dict = field(default_factory=dict)
    n_samples: int = 0
    seed: int = 0

    def __contains__(self, i):
        return i in self.layers

    def __getitem__(self, i):
        return self.layers[i]

    def indices(self):
        return sorted(self.layers)


class _FoldedLayer:
    def __init__(self, layer, w, b, precision="fp32"):
        self._l = layer
        self.weight = w
        self.bias = b
        self.bn = None
        self.precision = precision

    def __getattr__(self, k):
        return getattr(self._l, k)


class _Graph:
    def __init__(self, layers):
        self.layers = layers


def folded_graph(graph, precisions=None):
    """fold_all_bn + apply_plan (pm/model.py:183-193, 228-230) as a light view."""
    layers = []
    for l in graph.layers:
        if l.weight is None:
            layers.append(l)
            continue
        if l.bn is not None:
            w, b = fold_bn_arrays(l.weight, l.bias, l.bn.gamma, l.bn.beta, l.bn.mean, l.bn.var, l.bn.eps)
        else:
            w, b = l.weight, l.bias
        p = "fp32" if precisions is None else precisions.get(l.index, "fp32")
        layers.append(_FoldedLayer(l, w, b, p))
    return _Graph(layers)


def per_sample_ranges(graph, samples):
    """pm/calibration.py:106-128 -- FP32 folded forward, record each input's (min, max)."""
    fp32 = folded_graph(graph)
    out = []
    for pos, sample in enumerate(samples):
        ranges = {}

        def record(layer, x):
            lo, hi = minmax(x)
            if not (np.isfinite(lo) and np.isfinite(hi)):
                raise RuntimeError(
                    f"non-finite activation at layer {layer.index} ({layer.name!r}) "
                    f"on calibration sample {pos}"
                )
            ranges[layer.index] = (lo, hi)

        forward(fp32, sample, observe_fn=record)
        out.append(ranges)
    return out


def stats_from_ranges(graph, ranges, seed=0, per_channel_weights=False) -> Stats:
    """pm/calibration.py:131-154."""
    if not ranges:
        raise ValueError("calibration needs at least one sample")
    fp32 = folded_graph(graph)
    layers = {}
    for l in fp32.layers:
        if l.weight is None:
            continue
        lo, hi = math.inf, -math.inf
        for r in ranges:
            a, b = r[l.index]
            lo, hi = min(lo, a), max(hi, b)
        ws = weight_scales(l.weight, per_channel_weights)
        wqp = _PCQP(np.asarray(ws)) if per_channel_weights else _QP(float(ws))
        layers[l.index] = LayerStats(
            index=l.index, name=l.name, observer=_Obs(lo, hi, len(ranges)),
            act_qp=_QP(compute_scale(lo, hi)), weight_qp=wqp,
        )
    return Stats(layers=layers, n_samples=len(ranges), seed=seed)


def run_calibration(graph, samples, seed=0, per_channel_weights=False) -> Stats:
    """pm/calibration.py:157-165."""
    return stats_from_ranges(graph, per_sample_ranges(graph, samples), seed, per_channel_weights)


def planned_forward(graph, sample, stats, precisions: dict):
    """evaluate()'s per-frame body (pm/detector.py:320-325): fold, retag, forward."""
    return forward(folded_graph(graph, precisions), sample, stats=stats)


# ---------------------------------------------------------------------------
# decode: toy decode_and_nms (pm/detector.py:251-307) and the KITTI anchor top-k


def _sigmoid(x):
    """pm/detector.py:251-252."""
    return np.where(x >= 0, 1.0 / (1.0 + np.exp(-x)), np.exp(x) / (1.0 + np.exp(x)))


def _local_peaks(score_map):
    """pm/detector.py:255-263."""
    padded = np.pad(score_map, 1, constant_values=-np.inf)
    neighborhood = np.max(
        [padded[1 + di: padded.shape[0] - 1 + di, 1 + dj: padded.shape[1] - 1 + dj]
         for di in (-1, 0, 1) for dj in (-1, 0, 1)],
        axis=0,
    )
    return score_map >= neighborhood


def _iou(a, b):
    """pm/metrics.py:52-66 for one pair of (cx, cy, w, h) boxes."""
    ax1, ay1, ax2, ay2 = a[0] - a[2] / 2, a[1] - a[3] / 2, a[0] + a[2] / 2, a[1] + a[3] / 2
    bx1, by1, bx2, by2 = b[0] - b[2] / 2, b[1] - b[3] / 2, b[0] + b[2] / 2, b[1] + b[3] / 2
    iw = max(0.0, min(ax2, bx2) - max(ax1, bx1))
    ih = max(0.0, min(ay2, by2) - max(ay1, by1))
    inter = iw * ih
    union = a[2] * a[3] + b[2] * b[3] - inter
    return inter / union if union > 0 else 0.0


def decode_and_nms(cls_map, reg_map, field_size, base_size, score_thresh, iou_thresh):
    """pm/detector.py:266-307 -> list of (box[4] f64, class_id, score)."""
    logits = cls_map[0] if cls_map.ndim == 4 else cls_map
    reg = reg_map[0] if reg_map.ndim == 4 else reg_map
    n_classes, oh, ow = logits.shape
    cell_h = field_size / oh
    cell_w = field_size / ow
    scores = _sigmoid(logits.astype(np.float64))
    dets = []
    for cls in range(n_classes):
        peaks = _local_peaks(scores[cls])
        cand = []
        for i, j in np.argwhere(peaks):
            s = float(scores[cls, i, j])
            if s < score_thresh:
                continue
            dx, dy, dw, dh = (float(v) for v in reg[:, i, j])
            box = np.array([(j + 0.5 + dx) * cell_w, (i + 0.5 + dy) * cell_h,
                            base_size * math.exp(min(4.0, max(-4.0, dw))),
                            base_size * math.exp(min(4.0, max(-4.0, dh)))])
            cand.append((box, cls, s))
        cand.sort(key=lambda d: -d[2])
        kept = []
        for det in cand:
            if any(_iou(det[0], k[0]) >= iou_thresh for k in kept):
                continue
            kept.append(det)
        dets.extend(kept)
    return dets


def topk_anchor_order(cls_nchw: np.ndarray, k: int) -> np.ndarray:
    """KITTI extension: flat anchor index = (y*W + x)*A + a, ranked
    by f32 logit descending, ties to the lower index (SPEC.md:376 tie rule)."""
    logits = np.asarray(cls_nchw, np.float32)
    a_, h, w = logits.shape
    flat = logits.transpose(1, 2, 0).reshape(-1)
    idx = np.arange(flat.size)
    order = np.lexsort((idx, -flat.astype(np.float64)))
    return order[: min(k, flat.size)]


def decode_anchor_boxes(idx, box_nchw, dir_nchw, geom):
    """SECOND/PointPillars delta box coder (x,y,z,w,l,h,r) + direction bins in f32.

    Anchors: centre of output cell (x_min + (j+.5)*sx, y_min + (i+.5)*sy),
    z = anchor_z, size (w, l, h), yaw = rotations[a].  Boxes are compared with
    a tolerance (exp/sqrt rounding differs between libms); indices exactly.
    """
    A = len(geom.anchor_rotations)
    _, h, w = box_nchw.shape
    idx = np.asarray(idx, np.int64)
    cell = idx // A
    a = idx % A
    yy, xx = cell // w, cell % w
    f = np.float32
    deltas = box_nchw.reshape(A, 7, h, w)[a, :, yy, xx].astype(np.float32)  # [k, 7]
    dirs = dir_nchw.reshape(A, 2, h, w)[a, :, yy, xx].astype(np.float32)
    sx = f(geom.out_stride[0])
    sy = f(geom.out_stride[1])
    xa = f(geom.origin[0]) + (xx.astype(np.float32) + f(0.5)) * sx
    ya = f(geom.origin[1]) + (yy.astype(np.float32) + f(0.5)) * sy
    wa, la, ha = f(geom.anchor_size[0]), f(geom.anchor_size[1]), f(geom.anchor_size[2])
    za = f(geom.anchor_z) + ha / f(2.0)
    ra = np.asarray(geom.anchor_rotations, np.float32)[a]
    diag = np.sqrt(la * la + wa * wa).astype(np.float32)
    xg = deltas[:, 0] * diag + xa
    yg = deltas[:, 1] * diag + ya
    zg = deltas[:, 2] * ha + za
    wg = np.exp(deltas[:, 3]) * wa
    lg = np.exp(deltas[:, 4]) * la
    hg = np.exp(deltas[:, 5]) * ha
    rg = deltas[:, 6] + ra
    zg = zg - hg / f(2.0)
    label = (dirs[:, 1] > dirs[:, 0]).astype(np.int64)
    off = f(geom.dir_offset)
    period = f(np.pi)
    val = rg - off
    rot = val - np.floor(val / period) * period
    rg = rot + off + period * label.astype(np.float32)
    boxes = np.stack([xg, yg, zg, wg, lg, hg, rg], axis=1).astype(np.float32)
    return boxes, label


def decode_topk(cls_nchw, box_nchw, dir_nchw, geom, k):
    """Per-frame top-k anchors: (indices, f32 logits, f64 sigmoid scores, boxes, dir labels)."""
    order = topk_anchor_order(cls_nchw, k)
    A = len(geom.anchor_rotations)
    a_, h, w = cls_nchw.shape
    logits = np.asarray(cls_nchw, np.float32).transpose(1, 2, 0).reshape(-1)[order]
    scores = _sigmoid(logits.astype(np.float64))
    boxes, labels = decode_anchor_boxes(order, box_nchw, dir_nchw, geom)
    return order, logits, scores, boxes, labels
