"""Tensor types and the GPU dense kernels behind them (pm/tensor_ops.py counterpart).

``ConvParams`` and ``PillarSample`` are the reference's types (same fields,
validation and messages).  ``linear`` / ``conv2d`` run libpmx's implicit-GEMM
kernel in FP32 with the reference's shape errors; they exist for drop-in
completeness -- the engine (``engine.py``) calls the same kernel with the layer's
precision and fused epilogues.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N

__all__ = ["ConvParams", "PillarSample", "as_tensor", "conv2d", "linear"]


def as_tensor(values) -> np.ndarray:
    """Coerce to a C-contiguous float32 ndarray (pm/tensor_ops.py:25-27)."""
    return np.ascontiguousarray(values, dtype=np.float32)


@dataclass(frozen=True)
class ConvParams:
    """Stride/padding per spatial axis (pm/tensor_ops.py:34-57)."""

    stride: tuple[int, int] = (1, 1)
    padding: tuple[int, int] = (0, 0)

    def __post_init__(self):
        if any(s < 1 for s in self.stride):
            raise ValueError(f"stride must be positive, got {self.stride}")
        if any(p < 0 for p in self.padding):
            raise ValueError(f"padding must be non-negative, got {self.padding}")

    def out_size(self, in_hw: tuple[int, int], k_hw: tuple[int, int]) -> tuple[int, int]:
        out = []
        for size, k, s, p in zip(in_hw, k_hw, self.stride, self.padding):
            o = (size + 2 * p - k) // s + 1
            if o < 1:
                raise ValueError(
                    f"conv output extent {o} < 1 for input {size}, kernel {k}, stride {s}, padding {p}"
                )
            out.append(o)
        return out[0], out[1]


@dataclass(frozen=True)
class PillarSample:
    """One pillarized scene (pm/tensor_ops.py:60-77).

    features: [P, max_points, C] float32, zero-padded past each pillar's count
    point_mask: [P, max_points] bool
    coords: [P, 2] int (row, col), unique per pillar
    grid: (H, W)
    """

    features: np.ndarray
    point_mask: np.ndarray
    coords: np.ndarray
    grid: tuple[int, int]

    @property
    def num_pillars(self) -> int:
        return int(self.features.shape[0])


def _run_conv(x_nhwc, w_krsc, bias, desc_kw) -> "torch.Tensor":
    import torch

    lib = N.require_cuda()
    d = N.ConvDesc(**desc_kw)
    out = torch.empty((d.batch, d.out_h, d.out_w, d.out_c), dtype=torch.float32, device="cuda")
    outs, n = N.outs_array([N.Out(ptr=out.data_ptr(), scale=0.0, dtype=N.PMX_F32, c_stride=d.out_c,
                                  c_offset=0)])
    ws_bytes = lib.pmx_conv_workspace(C_ref(d))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    N.check(lib.pmx_conv(C_ref(d), x_nhwc.data_ptr(), w_krsc.data_ptr(), None, bias.data_ptr(), None, outs, n,
                         None, ws.data_ptr(), ws_bytes, N.stream_ptr()), "conv2d")
    return out


def C_ref(s):
    import ctypes

    return ctypes.byref(s)


def linear(x, weight, bias) -> np.ndarray:
    """x[..., Din] @ weight[Dout, Din].T + bias[Dout] (pm/tensor_ops.py:80-91), FP32 on the GPU."""
    import torch

    x = np.asarray(x, dtype=np.float32)
    if x.shape[-1] != weight.shape[1]:
        raise ValueError(f"linear input features {x.shape[-1]} != weight in-features {weight.shape[1]}")
    if bias.shape != (weight.shape[0],):
        raise ValueError(f"linear bias shape {bias.shape} != (out-features,) = ({weight.shape[0]},)")
    rows = int(np.prod(x.shape[:-1])) if x.ndim > 1 else 1
    din, dout = weight.shape[1], weight.shape[0]
    if rows == 0:
        return np.zeros(x.shape[:-1] + (dout,), np.float32)
    xd = torch.from_numpy(np.ascontiguousarray(x.reshape(rows, din))).cuda()
    wd = torch.from_numpy(np.ascontiguousarray(weight, np.float32)).cuda()
    bd = torch.from_numpy(np.ascontiguousarray(bias, np.float32)).cuda()
    out = _run_conv(xd, wd, bd, dict(kind=N.PMX_CONV2D, in_dtype=N.PMX_F32, batch=1, in_h=1, in_w=rows, in_c=din,
                                     in_c_stride=din, in_c_offset=0, out_c=dout, k_h=1, k_w=1, stride_h=1,
                                     stride_w=1, pad_h=0, pad_w=0, out_h=1, out_w=rows, relu=0))
    return out.cpu().numpy().reshape(x.shape[:-1] + (dout,))


def conv2d(x, weight, bias, params: ConvParams = ConvParams()) -> np.ndarray:
    """Cross-correlate x[N,C,H,W] with weight[F,C,kh,kw] + bias[F] (pm/tensor_ops.py:109-131)."""
    import torch

    x = np.asarray(x, dtype=np.float32)
    if x.ndim != 4 or weight.ndim != 4:
        raise ValueError(f"conv2d expects 4D input/weight, got {x.shape} and {weight.shape}")
    n, c, h, w = x.shape
    f, cw, kh, kw = weight.shape
    if c != cw:
        raise ValueError(f"conv2d input channels {c} != weight channels {cw}")
    if bias.shape != (f,):
        raise ValueError(f"conv2d bias shape {bias.shape} != ({f},)")
    ho, wo = params.out_size((h, w), (kh, kw))
    if n == 0:
        return np.zeros((0, f, ho, wo), np.float32)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda().permute(0, 2, 3, 1).contiguous()
    wd = torch.from_numpy(np.ascontiguousarray(weight.transpose(0, 2, 3, 1), np.float32)).cuda()
    bd = torch.from_numpy(np.ascontiguousarray(bias, np.float32)).cuda()
    out = _run_conv(xd, wd, bd, dict(kind=N.PMX_CONV2D, in_dtype=N.PMX_F32, batch=n, in_h=h, in_w=w, in_c=c,
                                     in_c_stride=c, in_c_offset=0, out_c=f, k_h=kh, k_w=kw,
                                     stride_h=params.stride[0], stride_w=params.stride[1],
                                     pad_h=params.padding[0], pad_w=params.padding[1], out_h=ho, out_w=wo,
                                     relu=0))
    return np.ascontiguousarray(out.permute(0, 3, 1, 2).cpu().numpy())
