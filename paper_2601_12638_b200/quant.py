"""Symmetric INT8 quantization, FP16 simulation and min/max observers (GPU-backed).

Same names, signatures, values and exceptions as the reference's
``pm/quant.py``; the element-wise math runs in libpmx's K1/K2 kernels
(``include/pmx.h``).  Host-side scalar parameter math (``compute_scale``,
dataclass validation) is the reference's own f64 formula, evaluated on the host
exactly like the reference does.

Arrays in, arrays out: numpy inputs come back as numpy (copied through the GPU);
``torch.Tensor`` CUDA inputs stay on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native as N

__all__ = [
    "DType",
    "FP16_MAX",
    "MinMaxObserver",
    "PerChannelQuantParams",
    "Q_MAX",
    "Q_MIN",
    "QuantParams",
    "compute_scale",
    "dequantize",
    "fake_quant",
    "fake_quant_per_channel",
    "fp16_roundtrip",
    "observe",
    "quantize",
    "weight_quant_params",
]

Q_MIN = -128
Q_MAX = 127
FP16_MAX = 65504.0


class DType(str, Enum):
    """Per-layer datatype tag (pm/quant.py:40-48)."""

    FP32 = "fp32"
    FP16 = "fp16"
    INT8 = "int8"

    def __str__(self) -> str:
        return self.value


@dataclass(frozen=True)
class QuantParams:
    """Symmetric per-tensor quantization parameters (pm/quant.py:51-64)."""

    scale: float
    zero_point: int = 0
    q_min: int = Q_MIN
    q_max: int = Q_MAX

    def __post_init__(self):
        if not math.isfinite(self.scale) or self.scale <= 0.0:
            raise ValueError(f"scale must be positive and finite, got {self.scale}")
        if self.zero_point != 0:
            raise ValueError("symmetric quantization requires zero_point == 0")


@dataclass(frozen=True)
class PerChannelQuantParams:
    """Per-output-channel weight scales, axis 0 (pm/quant.py:67-79)."""

    scales: np.ndarray
    q_min: int = Q_MIN
    q_max: int = Q_MAX

    def __post_init__(self):
        scales = np.asarray(self.scales, dtype=np.float64)
        if scales.ndim != 1 or not np.all(np.isfinite(scales)) or np.any(scales <= 0):
            raise ValueError("per-channel scales must be a 1D positive finite array")
        object.__setattr__(self, "scales", scales)

    def __eq__(self, other):
        return isinstance(other, PerChannelQuantParams) and np.array_equal(self.scales, other.scales)

    __hash__ = None


def compute_scale(x_min: float, x_max: float) -> QuantParams:
    """max(|x_min|, |x_max|) / 127; all-zero range -> 1.0 (pm/quant.py:82-95)."""
    if not (math.isfinite(x_min) and math.isfinite(x_max)):
        raise ValueError(f"non-finite calibration range ({x_min}, {x_max})")
    if x_min > x_max:
        raise ValueError(f"calibration range has min {x_min} > max {x_max}")
    max_abs = max(abs(x_min), abs(x_max))
    if max_abs == 0.0:
        return QuantParams(scale=1.0)
    return QuantParams(scale=max_abs / Q_MAX)


# ---------------------------------------------------------------------------
# device helpers


def _to_device(x, keep_f64: bool):
    """-> (contiguous CUDA tensor, was_host, original shape).  f64 inputs stay f64
    when ``keep_f64`` (the reference divides them in f64 without an f32 cast)."""
    import torch

    N.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.detach()
        want = torch.float64 if (keep_f64 and t.dtype == torch.float64) else torch.float32
        t = t.to(want)
        return t.contiguous().cuda(), False, tuple(t.shape)
    a = np.asarray(x)
    want = np.float64 if (keep_f64 and a.dtype != np.float32 and a.dtype != np.float16) else np.float32
    a = np.ascontiguousarray(a, dtype=want)
    return torch.from_numpy(a).cuda(), True, a.shape


def _to_device_f32(x):
    return _to_device(x, keep_f64=False)


def _back(t, as_numpy: bool, shape):
    if as_numpy:
        return t.cpu().numpy().reshape(shape)
    return t.reshape(shape)


def _code(t) -> int:
    import torch

    return N.PMX_F64 if t.dtype == torch.float64 else N.PMX_F32


def quantize(x, qp: QuantParams):
    """clamp(round_half_even(x / scale), -128, 127); scalar in, int out (pm/quant.py:98-103).

    f32 tensors: bit-exact with the reference's f64 divide through the K1
    guard-band kernel; f64 inputs are divided in f64 on the device."""
    import torch

    t, as_np, shape = _to_device(x, keep_f64=True)
    out = torch.empty(t.shape, dtype=torch.int32, device=t.device)
    N.check(N.load().pmx_quantize(t.data_ptr(), _code(t), t.numel(), float(qp.scale), out.data_ptr(),
                                  N.stream_ptr()), "quantize")
    if np.ndim(x) == 0 and not isinstance(x, torch.Tensor):
        return int(out.item())
    return _back(out, as_np, shape)


def dequantize(x_q, qp: QuantParams):
    """x_q * scale in f64 (pm/quant.py:106-111): host arithmetic on integer codes."""
    out = np.asarray(x_q, dtype=np.float64) * qp.scale
    if np.ndim(x_q) == 0:
        return float(out)
    return out


def fake_quant(t, qp: QuantParams):
    """Quantize-then-dequantize; f32 out, shape preserved (pm/quant.py:114-116)."""
    import torch

    d, as_np, shape = _to_device(t, keep_f64=True)
    out = torch.empty(d.shape, dtype=torch.float32, device=d.device)
    N.check(N.load().pmx_fake_quant(d.data_ptr(), _code(d), d.numel(), float(qp.scale), out.data_ptr(),
                                    N.stream_ptr()), "fake_quant")
    return _back(out, as_np, shape)


def weight_quant_params(weight, per_channel: bool = False):
    """Per-tensor (range includes 0) or per-output-channel params (pm/quant.py:119-133).

    Reductions over a one-shot weight tensor: host f64 like the reference (these
    are parameters, not activations)."""
    w = np.asarray(weight, dtype=np.float64)
    if not np.all(np.isfinite(w)):
        raise ValueError("weight tensor contains non-finite values")
    if not per_channel:
        return compute_scale(float(w.min(initial=0.0)), float(w.max(initial=0.0)))
    flat = w.reshape(w.shape[0], -1)
    max_abs = np.abs(flat).max(axis=1)
    scales = np.where(max_abs == 0.0, 1.0, max_abs / Q_MAX)
    return PerChannelQuantParams(scales=scales)


def weight_codes(weight, qp) -> "torch.Tensor":
    """int8 codes of a weight tensor on the device, per-row scales (K1 rows kernel)."""
    import torch

    d, _, shape = _to_device_f32(weight)
    rows = shape[0] if len(shape) else 1
    cols = d.numel() // max(rows, 1)
    if isinstance(qp, PerChannelQuantParams):
        sc = torch.from_numpy(np.asarray(qp.scales, np.float64)).cuda()
    else:
        sc = torch.full((rows,), float(qp.scale), dtype=torch.float64, device=d.device)
    codes = torch.empty(shape, dtype=torch.int8, device=d.device)
    N.check(N.load().pmx_quantize_rows(d.data_ptr(), rows, cols, sc.data_ptr(), codes.data_ptr(), None,
                                       N.stream_ptr()), "weight_codes")
    return codes


def fake_quant_per_channel(weight, qp: PerChannelQuantParams):
    """fake_quant with one scale per output channel, axis 0 (pm/quant.py:136-141)."""
    import torch

    d, as_np, shape = _to_device_f32(weight)
    rows = shape[0]
    cols = d.numel() // max(rows, 1)
    sc = torch.from_numpy(np.asarray(qp.scales, np.float64)).cuda()
    out = torch.empty_like(d)
    N.check(N.load().pmx_quantize_rows(d.data_ptr(), rows, cols, sc.data_ptr(), None, out.data_ptr(),
                                       N.stream_ptr()), "fake_quant_per_channel")
    return _back(out, as_np, shape)


def fp16_roundtrip(t):
    """Round to binary16 and back, saturating at +-65504 (pm/quant.py:144-147)."""
    import torch

    d, as_np, shape = _to_device_f32(t)
    out = torch.empty_like(d)
    N.check(N.load().pmx_fp16_roundtrip(d.data_ptr(), d.numel(), out.data_ptr(), None, N.stream_ptr()),
            "fp16_roundtrip")
    r = _back(out, as_np, shape)
    if as_np and np.ndim(t) == 0:
        return np.float32(r)
    return r


def to_fp16_bits(t) -> "torch.Tensor":
    """Saturating binary16 copy on the device (FP16 layer operands)."""
    import torch

    d, _, shape = _to_device_f32(t)
    out = torch.empty(shape, dtype=torch.float16, device=d.device)
    N.check(N.load().pmx_fp16_roundtrip(d.data_ptr(), d.numel(), None, out.data_ptr(), N.stream_ptr()),
            "to_fp16_bits")
    return out


def device_minmax(t) -> tuple[float, float]:
    """Exact (min, max) of a tensor through the K2 observer kernel."""
    import torch

    lib = N.require_cuda()
    if (isinstance(t, np.ndarray) and t.dtype == np.float64) or (
            isinstance(t, torch.Tensor) and t.dtype == torch.float64):
        d, _, _ = _to_device(t, keep_f64=True)
        keys = torch.empty(2, dtype=torch.int64, device="cuda")
        s = N.stream_ptr()
        N.check(lib.pmx_minmax_f64_init(keys.data_ptr(), s), "minmax_f64_init")
        N.check(lib.pmx_minmax_f64(d.data_ptr(), d.numel(), keys.data_ptr(), s), "minmax_f64")
        lo, hi = N.decode_keys64(keys.cpu().numpy().view(np.uint64))
        return float(lo), float(hi)
    if isinstance(t, torch.Tensor) and t.is_cuda:
        d = t.detach().contiguous()
        code = {torch.float32: N.PMX_F32, torch.float16: N.PMX_F16, torch.int8: N.PMX_I8}.get(d.dtype)
        if code is None:
            d = d.float()
            code = N.PMX_F32
    else:
        d, _, _ = _to_device_f32(t)
        code = N.PMX_F32
    keys = torch.empty(2, dtype=torch.int32, device="cuda")
    s = N.stream_ptr()
    N.check(lib.pmx_minmax_init(keys.data_ptr(), 1, s), "minmax_init")
    N.check(lib.pmx_minmax(d.data_ptr(), d.numel(), code, keys.data_ptr(), s), "minmax")
    lo, hi = N.decode_keys(keys.cpu().numpy().view(np.uint32))
    return float(lo), float(hi)


@dataclass(frozen=True)
class MinMaxObserver:
    """Running min/max; count == 0 is the empty sentinel (pm/quant.py:150-176)."""

    running_min: float = math.inf
    running_max: float = -math.inf
    count: int = 0

    @property
    def is_empty(self) -> bool:
        return self.count == 0

    def merge(self, other: "MinMaxObserver") -> "MinMaxObserver":
        if other.is_empty:
            return self
        if self.is_empty:
            return other
        return MinMaxObserver(
            running_min=min(self.running_min, other.running_min),
            running_max=max(self.running_max, other.running_max),
            count=self.count + other.count,
        )

    def quant_params(self) -> QuantParams:
        if self.is_empty:
            raise ValueError("cannot derive quant params from an empty observer")
        return compute_scale(self.running_min, self.running_max)


def observe(obs: MinMaxObserver, t) -> MinMaxObserver:
    """Widen the observer to cover every element of t (pm/quant.py:179-188); K2 kernel."""
    n = t.numel() if hasattr(t, "numel") else np.asarray(t).size
    if n == 0:
        return obs
    t_min, t_max = device_minmax(t)
    if not (math.isfinite(t_min) and math.isfinite(t_max)):
        raise ValueError("observed tensor contains non-finite values")
    return obs.merge(MinMaxObserver(running_min=t_min, running_max=t_max, count=1))
