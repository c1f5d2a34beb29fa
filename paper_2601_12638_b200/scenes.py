"""Pillarization entry points (pm/scenes.py:155-193 counterpart) on the GPU.

``pillarize(scene, grid, max_points_per_pillar, field_size)`` keeps the
reference signature and result (PillarSample with 5 features, pillars in
ascending (row, col) order, first-come truncation, no cap) but runs libpmx's K3
kernels.  ``pillarize_points`` is the KITTI-shaped variant (origin offset, 9
features, max-pillars cap) used by the engine.  The synthetic scene generator
and JSONL IO of the reference are out of scope.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import GridSpec
from .tensor_ops import PillarSample

__all__ = ["POINT_FEATURES", "Scene", "pillarize", "pillarize_points", "pillar_index"]

POINT_FEATURES = 5  # x, y, intensity, dx-to-pillar-mean, dy-to-pillar-mean


@dataclass(frozen=True)
class Scene:
    """Points [N, 3] as (x, y, intensity); boxes [M, 4] (pm/scenes.py:74-81)."""

    points: np.ndarray
    boxes: np.ndarray = None
    classes: np.ndarray = None
    difficulty: np.ndarray = None


def _run_pillarize(points4: np.ndarray, spec: GridSpec, n_features: int | None):
    """points4 [N, 4] f32 -> dict of device outputs (single frame)."""
    import torch

    lib = N.require_cuda()
    n = int(points4.shape[0])
    h, w = spec.grid
    pcap = spec.max_pillars if spec.max_pillars else h * w
    g = spec.to_c()
    pts = torch.from_numpy(np.ascontiguousarray(points4, np.float32)).cuda() if n else torch.zeros(
        (1, 4), dtype=torch.float32, device="cuda")
    offs = torch.tensor([0, n], dtype=torch.int64, device="cuda")
    coords = torch.empty((1, pcap, 2), dtype=torch.int32, device="cuda")
    counts = torch.empty((1, pcap), dtype=torch.int32, device="cuda")
    pt_idx = torch.empty((1, pcap, spec.max_points), dtype=torch.int32, device="cuda")
    n_pil = torch.zeros((1,), dtype=torch.int32, device="cuda")
    ws_bytes = lib.pmx_pillarize_workspace(ctypes.byref(g), 1, max(n, 1))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    s = N.stream_ptr()
    N.check(lib.pmx_pillarize(pts.data_ptr(), offs.data_ptr(), 1, max(n, 1), ctypes.byref(g), pcap,
                              coords.data_ptr(), counts.data_ptr(), pt_idx.data_ptr(), n_pil.data_ptr(),
                              ws.data_ptr(), ws_bytes, s), "pillarize")
    P = int(n_pil.item()) if n else 0
    out = {"coords": coords[0, :P], "counts": counts[0, :P], "pt_idx": pt_idx[0, :P], "n_pillars": P}
    if n_features is not None:
        feats = torch.zeros((1, max(P, 1), spec.max_points, n_features), dtype=torch.float32, device="cuda")
        mask = torch.zeros((1, max(P, 1), spec.max_points), dtype=torch.uint8, device="cuda")
        if P:
            N.check(lib.pmx_pillar_features(pts.data_ptr(), offs.data_ptr(), 1, ctypes.byref(g), max(P, 1),
                                            n_features, coords.data_ptr(), counts.data_ptr(), pt_idx.data_ptr(),
                                            n_pil.data_ptr(), feats.data_ptr(), mask.data_ptr(), s),
                    "pillar_features")
        out["features"] = feats[0, :P]
        out["mask"] = mask[0, :P]
    return out


def _sample(out, spec: GridSpec, n_features: int) -> PillarSample:
    P = out["n_pillars"]
    M = spec.max_points
    if P == 0:
        return PillarSample(features=np.zeros((0, M, n_features), np.float32),
                            point_mask=np.zeros((0, M), bool), coords=np.zeros((0, 2), np.int64),
                            grid=tuple(spec.grid))
    return PillarSample(features=out["features"].cpu().numpy(), point_mask=out["mask"].cpu().numpy().astype(bool),
                        coords=out["coords"].cpu().numpy().astype(np.int64), grid=tuple(spec.grid))


def pillarize(scene: Scene, grid: tuple[int, int], max_points_per_pillar: int, field_size: float) -> PillarSample:
    """Bucket points into grid cells and build padded per-pillar features (pm/scenes.py:155-193)."""
    h, w = grid
    if h < 1 or w < 1:
        raise ValueError(f"grid extents must be positive, got {grid}")
    pts = np.asarray(scene.points, np.float32)
    spec = GridSpec(grid=(h, w), origin=(0.0, 0.0), cell=(field_size / w, field_size / h),
                    max_points=max_points_per_pillar, max_pillars=None)
    if len(pts) == 0:
        return PillarSample(features=np.zeros((0, max_points_per_pillar, POINT_FEATURES), np.float32),
                            point_mask=np.zeros((0, max_points_per_pillar), bool),
                            coords=np.zeros((0, 2), np.int64), grid=grid)
    p4 = np.zeros((len(pts), 4), np.float32)
    p4[:, :3] = pts[:, :3]
    return _sample(_run_pillarize(p4, spec, POINT_FEATURES), spec, POINT_FEATURES)


def pillar_index(points: np.ndarray, spec: GridSpec) -> dict:
    """Integer pillarize outputs (coords, counts, pt_idx, n_pillars) as host arrays."""
    out = _run_pillarize(np.asarray(points, np.float32), spec, None)
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


def pillarize_points(points: np.ndarray, spec: GridSpec) -> PillarSample:
    """KITTI pillarize: [N, 4] (x, y, z, r) -> PillarSample with the 9 PointPillars features."""
    return _sample(_run_pillarize(np.asarray(points, np.float32), spec, 9), spec, 9)
