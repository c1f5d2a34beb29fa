"""Post-processing entry points: anchor decode + top-k on the GPU (K11).

The reference decodes its toy heads with local peaks + per-class NMS
(pm/detector.py:266-307); the KITTI heads of BASELINE.json need anchor
decoding instead, which the reference lacks.  This
follows the reference's conventions: deterministic ranking (f32 logit, then the
lower flat anchor index) and a SECOND delta box coder.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .engine import AnchorSpec

__all__ = ["decode_topk"]


def decode_topk(cls_map, box_map, dir_map, spec: AnchorSpec):
    """Top-k anchors of each frame from NCHW head maps ([B, A, H, W], [B, 7A, H, W], [B, 2A, H, W]).

    Returns dict of device tensors: idx [B,k] int32 (flat (y*W+x)*A+a), logit
    [B,k], boxes [B,k,7] (x, y, z, w, l, h, yaw), dir [B,k] int32.
    """
    import torch

    lib = N.require_cuda()

    def dev(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, np.float32))
        t = t.float().cuda()
        return t.unsqueeze(0) if t.dim() == 3 else t

    c, b, d = dev(cls_map), dev(box_map), dev(dir_map)
    A = len(spec.rotations)
    B, _, H, W = c.shape
    heads = torch.cat([c, b, d], dim=1).permute(0, 2, 3, 1).contiguous()  # NHWC [B, H, W, 10A]
    desc = spec.to_c()
    ws_bytes = lib.pmx_decode_workspace(ctypes.byref(desc), B, H, W)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    out = {
        "idx": torch.empty((B, spec.k), dtype=torch.int32, device="cuda"),
        "logit": torch.empty((B, spec.k), dtype=torch.float32, device="cuda"),
        "boxes": torch.empty((B, spec.k, 7), dtype=torch.float32, device="cuda"),
        "dir": torch.empty((B, spec.k), dtype=torch.int32, device="cuda"),
    }
    N.check(lib.pmx_decode_topk(ctypes.byref(desc), B, H, W, heads.data_ptr(), 10 * A, 0, A, 8 * A,
                                out["idx"].data_ptr(), out["logit"].data_ptr(), out["boxes"].data_ptr(),
                                out["dir"].data_ptr(), ws.data_ptr(), ws_bytes, N.stream_ptr()), "decode_topk")
    return out
