"""Post-processing entry points on the GPU.

* ``decode_and_nms`` -- the reference's own decode (pm/detector.py:266-307):
  f64 sigmoid scores, 3x3 local peaks, score threshold, per-class greedy NMS,
  returning ``Detection`` records (pm/metrics.py:35-49); kernel K11b
  ``pmx_decode_nms``.
* ``decode_topk`` -- the KITTI heads of BASELINE.json need anchor decoding,
  which the reference lacks; it follows the reference's
  conventions: deterministic ranking (f32 logit, then the lower flat anchor
  index) and a SECOND delta box coder (kernel K11).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import AnchorSpec

__all__ = ["Detection", "decode_and_nms", "decode_and_nms_batch", "decode_topk"]


@dataclass(frozen=True)
class Detection:
    """One predicted box (cx, cy, w, h) with class id and confidence (pm/metrics.py:35-49)."""

    box: np.ndarray
    class_id: int
    score: float

    def __post_init__(self):
        box = np.asarray(self.box, dtype=np.float64)
        if box.shape != (4,) or box[2] <= 0 or box[3] <= 0:
            raise ValueError(f"detection box must be (cx, cy, w, h) with positive extents, got {box}")
        if not np.isfinite(self.score):
            raise ValueError(f"detection score must be finite, got {self.score}")
        object.__setattr__(self, "box", box)


def _nms_desc(n_classes, oh, ow, cfg, score_thresh, iou_thresh):
    score_thresh = cfg.score_thresh if score_thresh is None else score_thresh
    iou_thresh = cfg.nms_iou if iou_thresh is None else iou_thresh
    if not (0.0 <= score_thresh <= 1.0 and 0.0 <= iou_thresh <= 1.0):
        raise ValueError(f"thresholds must lie in [0, 1], got {score_thresh}, {iou_thresh}")
    return N.NmsDesc(n_classes=n_classes, out_h=oh, out_w=ow, cell_w=cfg.field_size / ow,
                     cell_h=cfg.field_size / oh, base_size=float(cfg.base_size), score_thresh=float(score_thresh),
                     iou_thresh=float(iou_thresh))


def decode_and_nms_batch(cls_maps, reg_maps, cfg, score_thresh=None, iou_thresh=None):
    """Device-side batch form: cls [B, C, H, W], reg [B, 4, H, W] (torch CUDA tensors or
    arrays) -> (dets f64 [B, C, H*W, 5] = (cx, cy, w, h, score), n_dets int32 [B, C]),
    both on the device; frame b / class c keeps dets[b, c, :n_dets[b, c]] in order."""
    import torch

    lib = N.require_cuda()

    def dev(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, np.float32))
        return t.to(device="cuda", dtype=torch.float32).contiguous()

    c, r = dev(cls_maps), dev(reg_maps)
    if c.dim() != 4 or r.dim() != 4 or r.shape[1] != 4 or r.shape[0] != c.shape[0] or r.shape[2:] != c.shape[2:]:
        raise ValueError(f"expected cls [B, C, H, W] and reg [B, 4, H, W], got {tuple(c.shape)}, {tuple(r.shape)}")
    B, C, H, W = c.shape
    d = _nms_desc(C, H, W, cfg, score_thresh, iou_thresh)
    dets = torch.empty((B, C, H * W, 5), dtype=torch.float64, device="cuda")
    n = torch.zeros((B, C), dtype=torch.int32, device="cuda")
    N.check(lib.pmx_decode_nms(ctypes.byref(d), B, c.data_ptr(), r.data_ptr(), dets.data_ptr(), n.data_ptr(),
                               N.stream_ptr()), "decode_and_nms")
    return dets, n


def decode_and_nms(cls_map, reg_map, cfg, score_thresh=None, iou_thresh=None) -> list[Detection]:
    """pm/detector.py:266-307 on the GPU: cls [1, C, H, W] or [C, H, W] logits, reg the
    matching [.., 4, H, W] deltas; ``cfg`` supplies field_size, base_size, score_thresh and
    nms_iou (the reference's DetectorConfig, or any object with those attributes).
    Returns the class-major list of kept detections."""
    logits = np.asarray(cls_map)
    reg = np.asarray(reg_map)
    logits = logits[0] if logits.ndim == 4 else logits
    reg = reg[0] if reg.ndim == 4 else reg
    dets, n = decode_and_nms_batch(logits[None], reg[None], cfg, score_thresh, iou_thresh)
    dets, n = dets[0].cpu().numpy(), n[0].cpu().numpy()
    out = []
    for cls in range(dets.shape[0]):
        for row in dets[cls, : int(n[cls])]:
            out.append(Detection(box=row[:4].copy(), class_id=cls, score=float(row[4])))
    return out


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
