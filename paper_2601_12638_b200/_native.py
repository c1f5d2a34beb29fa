"""ctypes binding of libpmx.so (include/pmx.h) -- the only way the package reaches the GPU.

There is no CPU fallback: importing works without a GPU (so the CPU test tier
can check the library and its exports), but every compute entry point calls
``require_cuda()`` and raises if the CUDA device or the shared library is
missing.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["PMX_LIB"]) if os.environ.get("PMX_LIB") else PKG / "libpmx.so"  # PMX_LIB: A/B builds

PMX_OK, PMX_ERR_INVALID, PMX_ERR_CUDA, PMX_ERR_UNSUPPORTED = 0, 1, 2, 3
PMX_F32, PMX_F16, PMX_I8, PMX_F64, PMX_F32X2 = 0, 1, 2, 3, 4
PMX_CONV2D, PMX_DECONV2D = 0, 1
PMX_PFN_FROM_POINTS9, PMX_PFN_FROM_FEATURES = 0, 1
PMX_MAX_OUTS = 3

DTYPE_CODE = {"fp32": PMX_F32, "fp16": PMX_F16, "int8": PMX_I8}


class Grid(C.Structure):
    _fields_ = [("grid_h", C.c_int32), ("grid_w", C.c_int32), ("max_points", C.c_int32),
                ("max_pillars", C.c_int32), ("x_min", C.c_float), ("y_min", C.c_float),
                ("cell_w", C.c_float), ("cell_h", C.c_float)]


class Out(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("scale", C.c_double), ("dtype", C.c_int32),
                ("c_stride", C.c_int32), ("c_offset", C.c_int32), ("_reserved", C.c_int32)]


class PfnDesc(C.Structure):
    _fields_ = [("source", C.c_int32), ("in_dtype", C.c_int32), ("n_features", C.c_int32),
                ("channels", C.c_int32), ("max_points", C.c_int32), ("relu", C.c_int32),
                ("in_scale", C.c_double)]


class ConvDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "in_dtype", "batch", "in_h", "in_w", "in_c", "in_c_stride", "in_c_offset", "out_c",
        "k_h", "k_w", "stride_h", "stride_w", "pad_h", "pad_w", "out_h", "out_w", "relu")]


class AnchorDesc(C.Structure):
    _fields_ = [("n_anchors", C.c_int32), ("k", C.c_int32), ("x_min", C.c_float), ("y_min", C.c_float),
                ("stride_x", C.c_float), ("stride_y", C.c_float), ("anchor_z", C.c_float),
                ("anchor_w", C.c_float), ("anchor_l", C.c_float), ("anchor_h", C.c_float),
                ("rotations", C.c_float * 4), ("dir_offset", C.c_float), ("_pad", C.c_float)]


class NmsDesc(C.Structure):
    _fields_ = [("n_classes", C.c_int32), ("out_h", C.c_int32), ("out_w", C.c_int32), ("_pad", C.c_int32),
                ("cell_w", C.c_double), ("cell_h", C.c_double), ("base_size", C.c_double),
                ("score_thresh", C.c_double), ("iou_thresh", C.c_double)]


class HeadFuse(C.Structure):
    _fields_ = [("w_codes", C.c_void_p), ("n_heads", C.c_int32), ("stage", C.c_int32), ("in_scale", C.c_double),
                ("partial", C.c_void_p), ("heads", C.c_void_p), ("heads_c_stride", C.c_int32), ("part_stride", C.c_int32),
                ("head_alpha", C.c_void_p), ("head_bias", C.c_void_p)]


P = C.c_void_p
I32, I64, F64, SZ = C.c_int32, C.c_int64, C.c_double, C.c_size_t

# name -> (restype, argtypes); mirrors include/pmx.h one to one
SIGNATURES = {
    "pmx_last_error": (C.c_char_p, []),
    "pmx_abi_version": (I32, []),
    "pmx_conv_backend": (C.c_char_p, [I32, I32]),
    "pmx_quantize": (I32, [P, I32, I64, F64, P, P]),
    "pmx_fake_quant": (I32, [P, I32, I64, F64, P, P]),
    "pmx_quantize_rows": (I32, [P, I64, I64, P, P, P, P]),
    "pmx_fp16_roundtrip": (I32, [P, I64, P, P, P]),
    "pmx_minmax_init": (I32, [P, I64, P]),
    "pmx_minmax": (I32, [P, I64, I32, P, P]),
    "pmx_minmax_f64_init": (I32, [P, P]),
    "pmx_minmax_f64": (I32, [P, I64, P, P]),
    "pmx_pillarize_workspace": (SZ, [C.POINTER(Grid), I32, I64]),
    "pmx_pillarize": (I32, [P, P, I32, I64, C.POINTER(Grid), I32, P, P, P, P, P, SZ, P]),
    "pmx_pillar_features": (I32, [P, P, I32, C.POINTER(Grid), I32, I32, P, P, P, P, P, P, P]),
    "pmx_pfn_scatter": (I32, [C.POINTER(PfnDesc), C.POINTER(Grid), I32, I32, P, P, P, P, P, P, P, P, P, P,
                              P, P, C.POINTER(Out), I32, P, P, P]),
    "pmx_pfn_pillars": (I32, [C.POINTER(PfnDesc), C.POINTER(Grid), I32, I32, P, P, P, P, P, P, P, P, P, P,
                              P, P, C.POINTER(Out), I32, P, P, P]),
    "pmx_pillarize_cell_map": (P, [C.POINTER(Grid), I32, I64, P]),
    "pmx_conv_gather_supported": (I32, [C.POINTER(ConvDesc)]),
    "pmx_conv_gather": (I32, [C.POINTER(ConvDesc), P, P, I32, P, P, P, P, C.POINTER(Out), I32, P, P]),
    "pmx_conv_workspace": (SZ, [C.POINTER(ConvDesc)]),
    "pmx_conv_tc_supported": (I32, [C.POINTER(ConvDesc)]),
    "pmx_deconv_heads_supported": (I32, [C.POINTER(ConvDesc)]),
    "pmx_deconv_heads": (I32, [C.POINTER(ConvDesc), P, P, P, P, C.POINTER(HeadFuse), P]),
    "pmx_conv": (I32, [C.POINTER(ConvDesc), P, P, P, P, P, C.POINTER(Out), I32, P, P, SZ, P]),
    "pmx_set_conv_backend": (None, [I32]),
    "pmx_debug_trace": (None, [P]),
    "pmx_debug_timeline": (None, [P]),
    "pmx_upsample2x": (I32, [P, I32, I32, I32, I32, I32, P, P]),
    "pmx_cast_out": (I32, [P, I64, I32, C.POINTER(Out), I32, P, P]),
    "pmx_decode_workspace": (SZ, [C.POINTER(AnchorDesc), I32, I32, I32]),
    "pmx_decode_topk": (I32, [C.POINTER(AnchorDesc), I32, I32, I32, P, I32, I32, I32, I32, P, P, P, P, P, SZ,
                              P]),
    "pmx_decode_nms": (I32, [C.POINTER(NmsDesc), I32, P, P, P, P, P]),
    "pmx_pack_topk_records": (I32, [I32, I32, P, P, P, P, P, P]),
    "pmx_zero": (I32, [P, SZ, P]),
    "pmx_sq_err_workspace": (SZ, []),
    "pmx_sq_err": (I32, [P, P, I64, P, P, SZ, P]),
    # QAT (train.cu)
    "pmx_train_conv_fwd": (I32, [C.POINTER(ConvDesc), P, P, P, P, P]),
    "pmx_train_conv_dgrad": (I32, [C.POINTER(ConvDesc), P, P, P, P]),
    "pmx_train_conv_wgrad": (I32, [C.POINTER(ConvDesc), P, P, P, P, P]),
    "pmx_train_relu": (I32, [P, I64, P, P]),
    "pmx_train_relu_bwd": (I32, [P, P, I64, P, P]),
    "pmx_train_ste": (I32, [P, I64, F64, I32, I32, P, P, P]),
    "pmx_train_ste_rows": (I32, [P, I64, I64, P, I32, I32, P, P, P]),
    "pmx_train_maxpool": (I32, [P, P, I64, I32, I32, P, P, P]),
    "pmx_train_maxpool_bwd": (I32, [P, P, I64, I32, I32, P, P]),
    "pmx_train_scatter": (I32, [P, P, I64, I32, I32, P, P]),
    "pmx_train_scatter_bwd": (I32, [P, P, I64, I32, I32, P, P]),
    "pmx_train_upsample2x_bwd": (I32, [P, I32, I32, I32, I32, P, P]),
    "pmx_train_add": (I32, [P, P, I64, P, P]),
    "pmx_train_copy_channels": (I32, [P, I64, I32, I32, I32, P, I32, I32, P]),
    "pmx_train_reduce_workspace": (SZ, []),
    "pmx_train_detection_loss": (I32, [P, P, P, P, P, P, I64, I32, I32, F64, F64, F64, F64, P, P, P, P, P]),
    "pmx_train_mse_loss": (I32, [P, P, I64, P, P, P, P]),
    "pmx_train_sumsq": (I32, [P, I64, C.c_float, P, P, P]),
    "pmx_train_sgd": (I32, [P, P, I64, C.c_float, C.c_float, C.c_float, P, P]),
}

_LIB = None


def header_symbols() -> list[str]:
    """Function names declared in include/pmx.h (for the export check)."""
    import re

    text = (PKG.parent / "include" / "pmx.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(pmx_\w+)\s*\(", text, flags=re.M)))


def load(path: Path | None = None):
    """Load libpmx.so (building it in-tree when the sources are newer and nvcc exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    lib_path = Path(path) if path else LIB_PATH
    if path is None and os.environ.get("PMX_NO_BUILD") != "1":
        try:
            from . import _build

            if not _build.up_to_date():
                _build.build()
        except Exception as exc:  # building is best effort; a stale .so still loads
            if not lib_path.exists():
                raise RuntimeError(f"libpmx.so is missing and could not be built: {exc}") from exc
    if not lib_path.exists():
        raise RuntimeError(f"libpmx.so not found at {lib_path}; run __graft_entry__.build()")
    lib = C.CDLL(str(lib_path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2601_12638_b200 needs a CUDA device: the engine has no CPU path")
    return load()


class PmxError(RuntimeError):
    pass


def check(status: int, what: str = "pmx"):
    if status == PMX_OK:
        return
    msg = (load().pmx_last_error() or b"").decode(errors="replace")
    if status == PMX_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise PmxError(f"{what} failed ({status}): {msg}")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def outs_array(outs) -> tuple:
    arr = (Out * PMX_MAX_OUTS)()
    for i, o in enumerate(outs):
        arr[i] = o
    return arr, len(outs)


def decode_keys64(keys: np.ndarray) -> np.ndarray:
    """f64 observer keys [..., 2] uint64 -> float64 (min, max)."""
    k = np.asarray(keys, dtype=np.uint64)
    top = np.uint64(0x8000000000000000)
    neg = (k & top) == 0
    bits = np.where(neg, ~k, k & ~top).astype(np.uint64)
    return bits.view(np.float64)


def decode_keys(keys: np.ndarray) -> np.ndarray:
    """Observer keys [..., 2] uint32 -> float32 (min, max) (see pmx.h K2)."""
    k = np.asarray(keys, dtype=np.uint32)
    neg = (k & 0x80000000) == 0
    bits = np.where(neg, ~k, k & 0x7FFFFFFF).astype(np.uint32)
    return bits.view(np.float32)
