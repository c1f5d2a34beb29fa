"""KITTI-shaped PointPillars: geometry, seeded weights, synthetic frames, and the engine.

The reference's only model is a 16x16 toy (pm/detector.py:96-210); BASELINE.json
names the KITTI PointPillars instead.  This module
builds that network as a ``ModelGraph`` with the reference's conventions
(He-normal init std sqrt(2/fan_in), BN gamma~U(.8,1.2), beta~N(0,.05),
mu~N(0,.1), eps 1e-5, zero biases, pm/detector.py:86-107) and BASELINE's
var~U(0.5,1.5) override.  Layer indices follow the paper's Table II
(PAPER.md:345-389): 1 PFN, 2-5 blocks.0, 6-11 blocks.1, 12-17 blocks.2,
18-20 deblocks, 21 conv_dir_cls, 22 conv_reg, 23 conv_cls.

Design choices where the reference is silent:
deconv weights [Cout, Cin, k, k] with fan_in = Cin*k*k; heads
Kaiming with zero bias (App. B.6); anchors: car (w, l, h) = (1.6, 3.9, 1.56),
z = -1.78, yaw {0, pi/2}, centred on the 0.32 m output cells.
"""

from __future__ import annotations

import os

import math
from dataclasses import dataclass, field

import numpy as np

from .engine import AnchorSpec, CompiledGraph, GridSpec
from .model import BatchNorm, LayerSpec, ModelGraph, PrecisionPlan, apply_plan, fold_all_bn, parse_plan_label
from .tensor_ops import ConvParams

__all__ = ["PointPillarsConfig", "build_pointpillars", "make_frame", "make_frames", "PointPillarsEngine",
           "PipelinedEngine",
           "MIXED_PLAN_LABEL", "HEADS"]

# BASELINE config 3: first backbone conv + the three deconvs in FP16
MIXED_PLAN_LABEL = "FP16: 2,18,19,20"
HEADS = ("bbox_head.conv_dir_cls", "bbox_head.conv_reg", "bbox_head.conv_cls")


@dataclass(frozen=True)
class PointPillarsConfig:
    """KITTI car PointPillars geometry (BASELINE.json configs)."""

    x_range: tuple[float, float] = (0.0, 69.12)
    y_range: tuple[float, float] = (-39.68, 39.68)
    z_range: tuple[float, float] = (-3.0, 1.0)
    cell: tuple[float, float] = (0.16, 0.16)
    grid: tuple[int, int] = (496, 432)          # rows (y), cols (x)
    max_points: int = 32
    max_pillars: int = 12000
    pfn_channels: int = 64
    block_channels: tuple[int, int, int] = (64, 128, 256)
    block_convs: tuple[int, int, int] = (4, 6, 6)
    block_strides: tuple[int, int, int] = (2, 2, 2)
    upsample_strides: tuple[int, int, int] = (1, 2, 4)
    neck_channels: int = 128
    rotations: tuple[float, ...] = (0.0, 1.5707963)
    anchor_size: tuple[float, float, float] = (1.6, 3.9, 1.56)  # (w, l, h)
    anchor_z: float = -1.78
    dir_offset: float = 0.78539
    topk: int = 100

    @property
    def n_anchors(self) -> int:
        return len(self.rotations)

    @property
    def out_grid(self) -> tuple[int, int]:
        s = self.block_strides[0] // self.upsample_strides[0]
        return self.grid[0] // s, self.grid[1] // s

    @property
    def out_stride(self) -> tuple[float, float]:
        oh, ow = self.out_grid
        return ((self.x_range[1] - self.x_range[0]) / ow, (self.y_range[1] - self.y_range[0]) / oh)

    def grid_spec(self) -> GridSpec:
        return GridSpec(grid=self.grid, origin=(self.x_range[0], self.y_range[0]), cell=self.cell,
                        max_points=self.max_points, max_pillars=self.max_pillars)

    def anchor_spec(self) -> AnchorSpec:
        return AnchorSpec(k=self.topk, origin=(self.x_range[0], self.y_range[0]), out_stride=self.out_stride,
                          anchor_z=self.anchor_z, anchor_size=self.anchor_size, rotations=self.rotations,
                          dir_offset=self.dir_offset, cls_head=HEADS[2], box_head=HEADS[1], dir_head=HEADS[0])

    @staticmethod
    def small(grid=(64, 48), max_pillars=1500, **kw) -> "PointPillarsConfig":
        """Same network on a smaller grid (parity tests the CPU oracle finishes in seconds)."""
        h, w = grid
        return PointPillarsConfig(x_range=(0.0, w * 0.16), y_range=(-h * 0.08, h * 0.08), grid=grid,
                                  max_pillars=max_pillars, **kw)


def _bn(c: int, rng: np.random.Generator) -> BatchNorm:
    """pm/detector.py:86-93 with BASELINE's var ~ U(0.5, 1.5)."""
    return BatchNorm(
        gamma=rng.uniform(0.8, 1.2, size=c).astype(np.float32),
        beta=rng.normal(scale=0.05, size=c).astype(np.float32),
        mean=rng.normal(scale=0.1, size=c).astype(np.float32),
        var=rng.uniform(0.5, 1.5, size=c).astype(np.float32),
        eps=1e-5,
    )


def build_pointpillars(cfg: PointPillarsConfig = PointPillarsConfig(), seed: int = 0) -> ModelGraph:
    """Seeded random-init KITTI PointPillars (23 indexed layers) as a DAG ModelGraph."""
    rng = np.random.default_rng(seed)

    def kaiming(shape, fan_in):
        return rng.normal(scale=math.sqrt(2.0 / fan_in), size=shape).astype(np.float32)

    layers: list[LayerSpec] = []
    idx = 1
    c = cfg.pfn_channels
    layers.append(LayerSpec(name="voxel_encoder.pfn_layers.0.linear", kind="linear", index=idx,
                            weight=kaiming((c, 9), 9), bias=np.zeros(c, np.float32), bn=_bn(c, rng), relu=True))
    idx += 1
    layers.append(LayerSpec(name="voxel_encoder.maxpool", kind="maxpool"))
    layers.append(LayerSpec(name="middle_encoder.scatter", kind="scatter", grid=cfg.grid))
    cin = c
    block_out = []
    prev = "middle_encoder.scatter"
    for b, (cout, n, s) in enumerate(zip(cfg.block_channels, cfg.block_convs, cfg.block_strides)):
        for j in range(n):
            name = f"backbone.blocks.{b}.{3 * j}"
            layers.append(LayerSpec(
                name=name, kind="conv2d", index=idx, weight=kaiming((cout, cin, 3, 3), cin * 9),
                bias=np.zeros(cout, np.float32), bn=_bn(cout, rng), relu=True,
                conv=ConvParams(stride=(s, s) if j == 0 else (1, 1), padding=(1, 1)),
                inputs=(prev,) if j == 0 else None))
            idx += 1
            cin = cout
            prev = name
        block_out.append(prev)
    neck = []
    for b, (src, up) in enumerate(zip(block_out, cfg.upsample_strides)):
        cin_b = cfg.block_channels[b]
        name = f"neck.deblocks.{b}.0"
        layers.append(LayerSpec(
            name=name, kind="deconv2d", index=idx,
            weight=kaiming((cfg.neck_channels, cin_b, up, up), cin_b * up * up),
            bias=np.zeros(cfg.neck_channels, np.float32), bn=_bn(cfg.neck_channels, rng), relu=True,
            conv=ConvParams(stride=(up, up)), inputs=(src,)))
        idx += 1
        neck.append(name)
    layers.append(LayerSpec(name="neck.concat", kind="concat", inputs=tuple(neck)))
    ccat = cfg.neck_channels * len(neck)
    A = cfg.n_anchors
    for name, cout in ((HEADS[0], 2 * A), (HEADS[1], 7 * A), (HEADS[2], A)):
        layers.append(LayerSpec(name=name, kind="conv2d", index=idx, weight=kaiming((cout, ccat, 1, 1), ccat),
                                bias=np.zeros(cout, np.float32), conv=ConvParams(), is_head=True))
        idx += 1
    meta = {"model": "pointpillars-kitti-car", "seed": seed,
            "grid": list(cfg.grid), "max_pillars": cfg.max_pillars}
    return ModelGraph(layers=tuple(layers), meta=meta)


def make_frame(n_points: int, seed: int, cfg: PointPillarsConfig = PointPillarsConfig(),
               outlier_frac: float = 0.0) -> np.ndarray:
    """Seeded synthetic KITTI-shaped frame [N, 4] f32 (x, y, z, r) -- BASELINE.json configs.

    x ~ U[x_range), y ~ U[y_range), z = clip(N(-1.6, 0.4), -3, 1), r ~ U[0, 1);
    ``outlier_frac`` of the points (config 2: 1%) get r = 1 and z at a range limit.
    """
    rng = np.random.default_rng(seed)
    x = rng.uniform(cfg.x_range[0], cfg.x_range[1], n_points)
    y = rng.uniform(cfg.y_range[0], cfg.y_range[1], n_points)
    z = np.clip(rng.normal(-1.6, 0.4, n_points), cfg.z_range[0], cfg.z_range[1])
    r = rng.uniform(0.0, 1.0, n_points)
    n_out = int(round(outlier_frac * n_points))
    if n_out:
        pick = rng.choice(n_points, size=n_out, replace=False)
        r[pick] = 1.0
        z[pick] = rng.choice(np.array([cfg.z_range[0], cfg.z_range[1]]), size=n_out)
    return np.stack([x, y, z, r], axis=1).astype(np.float32)


def make_frames(n_frames: int, seed: int, cfg: PointPillarsConfig = PointPillarsConfig(),
                n_range: tuple[int, int] = (60000, 150000), outlier_frac: float = 0.0) -> list[np.ndarray]:
    """Config-4 style batch: per-frame point counts ~ U{n_range} (seeded)."""
    rng = np.random.default_rng(seed)
    counts = rng.integers(n_range[0], n_range[1] + 1, size=n_frames)
    return [make_frame(int(n), seed * 100003 + i, cfg, outlier_frac) for i, n in enumerate(counts)]


class PointPillarsEngine:
    """pillarize -> forward(plan) -> decode for a fixed batch, captured as one CUDA graph.

    ``stats`` are the calibration stats (required for INT8 layers); ``plan`` a
    PrecisionPlan or a label like "FP16: 2,18,19,20".  Inputs go through
    ``load_points`` (H2D into static buffers); outputs stay on the device.
    """

    def __init__(self, graph: ModelGraph, plan, stats=None, cfg: PointPillarsConfig = PointPillarsConfig(),
                 batch: int = 1, max_points_per_frame: int = 150000, observe: bool = False,
                 decode: bool = True, fold: bool = True):
        if isinstance(plan, str):
            plan = parse_plan_label(plan)
        self.plan = plan or PrecisionPlan()
        g = fold_all_bn(graph) if fold else graph
        self.graph = apply_plan(g, self.plan)
        self.cfg = cfg
        self.batch = batch
        self.nmax = max_points_per_frame
        self.cg = CompiledGraph(self.graph, stats, source="points", batch=batch, grid=cfg.grid_spec(),
                                pcap=cfg.max_pillars, max_points_per_frame=max_points_per_frame, observe=observe,
                                anchors=cfg.anchor_spec() if decode else None)

    def load_points(self, frames, stream=None, pinned: bool = False):
        """Copy frames (list of [N_i, 4] f32 arrays or one host tensor + offsets) into the engine."""
        import torch

        if len(frames) != self.batch:
            raise ValueError(f"engine compiled for batch {self.batch}, got {len(frames)} frames")
        counts = [len(f) for f in frames]
        if max(counts) > self.nmax:
            raise ValueError(f"frame with {max(counts)} points exceeds max_points_per_frame {self.nmax}")
        offs = np.zeros(self.batch + 1, np.int64)
        offs[1:] = np.cumsum(counts)
        host = torch.from_numpy(np.concatenate(frames, axis=0) if frames else np.zeros((0, 4), np.float32))
        if pinned:
            host = host.pin_memory()
        self.cg.points[: offs[-1]].copy_(host, non_blocking=pinned)
        self.cg.offsets.copy_(torch.from_numpy(offs), non_blocking=False)
        return offs

    def run(self, stream=None):
        if self.cg.graph_exec is not None:
            self.cg.replay()
        else:
            self.cg.launch(stream)

    def capture(self):
        return self.cg.capture()

    def heads(self) -> dict:
        return {h: self.cg.head_output(h) for h in HEADS}

    def heads_nchw(self) -> dict:
        return {h: t.permute(0, 3, 1, 2).contiguous() for h, t in self.heads().items()}

    def topk(self) -> dict:
        cg = self.cg
        return {"idx": cg.topk_idx, "logit": cg.topk_logit, "boxes": cg.topk_boxes, "dir": cg.topk_dir}

    def pillars(self) -> dict:
        cg = self.cg
        return {"coords": cg.coords, "counts": cg.counts, "pt_idx": cg.pt_idx, "n_pillars": cg.n_pillars}


class PipelinedEngine:
    """Host-to-device streaming around a PointPillarsEngine: two input slots (points +
    frame offsets) with one captured CUDA graph each; while the graph of batch i runs,
    the pinned-host copy of batch i+1 lands in the other slot on an H2D stream and the
    top-k records of batch i-1 go back on a D2H stream (the copy engines overlap the
    SMs).  Every batch's H2D and D2H still happen.

    With a second engine (``eng2``, same graph / plan / stats / batch, its own
    activation buffers) slot 1 runs on that engine and each slot replays on its own
    compute stream, so consecutive batches overlap on the SMs as well (one kernel's
    tail and the next kernel's launch of one batch are filled by the other's)."""

    def __init__(self, eng: "PointPillarsEngine", eng2: "PointPillarsEngine | None" = None):
        import torch

        self.eng = eng
        self.engines = [eng, eng2 if eng2 is not None else eng]
        if eng2 is not None and (eng2.batch != eng.batch or eng2.nmax != eng.nmax):
            raise ValueError("the two engines of a PipelinedEngine need the same batch and point capacity")
        self.slots, self.graphs = [], []
        # per slot: (front graph reading the input slot, rest) or None -- the next H2D into a
        # slot then waits only for the front part (pillarize + PFN) of the batch before
        self.split = []
        for k, e in enumerate(self.engines):
            cg = e.cg
            # a shared engine's slot 1 starts as a copy of slot 0 (capture() warms up on whatever
            # the slot holds); each slot's graph writes its own top-k records buffer (read back D2H)
            rec0 = getattr(cg, "records", None)
            if k == 1 and eng2 is None:
                pts, offs = cg.points.clone(), cg.offsets.clone()
                rec = None if rec0 is None else rec0.clone()
                keep = (cg.points, cg.offsets, rec0)
                cg.points, cg.offsets = pts, offs
                if rec is not None:
                    cg.records = rec
                self.graphs.append(cg.capture())
                self.split.append(cg.capture_split())
                cg.points, cg.offsets = keep[0], keep[1]
                if rec0 is not None:
                    cg.records = rec0
                cg.graph_exec = self.graphs[0]
                self.slots.append((pts, offs, rec))
            else:
                self.graphs.append(cg.capture())
                self.split.append(cg.capture_split())
                self.slots.append((cg.points, cg.offsets, rec0))
        self.h2d = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()
        self.comp = [None, torch.cuda.Stream() if eng2 is not None else None]
        self.copied = [torch.cuda.Event(), torch.cuda.Event()]
        self.done = [torch.cuda.Event(), torch.cuda.Event()]
        self.fetched = [torch.cuda.Event(), torch.cuda.Event()]
        self.read = [torch.cuda.Event(), torch.cuda.Event()]  # the slot's points / offsets consumed
        if any(sp is None for sp in self.split) or os.environ.get("PMX_PIPE_SPLIT") == "0":  # (A/B runs)
            self.split = [None, None]

    def _upload(self, i: int, host_points, host_offsets):
        import torch

        slot = i % 2
        pts, offs, _ = self.slots[slot]
        with torch.cuda.stream(self.h2d):
            if i >= 2:
                # batch i-2 finished reading this slot (split graphs: its front part)
                self.h2d.wait_event(self.read[slot] if self.split[slot] is not None else self.done[slot])
            pts[: host_points.shape[0]].copy_(host_points, non_blocking=True)
            offs.copy_(host_offsets, non_blocking=True)
            self.copied[slot].record(self.h2d)

    def run(self, batches, host_out, pack=None):
        """batches: list of (pinned points [N, 4] f32, pinned offsets [B + 1] i64);
        host_out: list of pinned tensors receiving each batch's top-k records [B, k, 10]
        (written inside the graph), or pack(topk) when a pack function is given."""
        import torch

        main = torch.cuda.current_stream()
        comps = [main if c is None else c for c in self.comp]
        start = torch.cuda.Event()
        start.record(main)
        for c in comps:
            if c is not main:
                c.wait_event(start)
        n = len(batches)
        if n == 0:
            return
        self._upload(0, *batches[0])
        for i in range(n):
            slot = i % 2
            comp = comps[slot]
            if i + 1 < n:
                self._upload(i + 1, *batches[i + 1])
            comp.wait_event(self.copied[slot])
            if i >= 2:
                # batch i-2's D2H copy (d2h stream) must have finished reading this slot's
                # records buffer before the graph rewrites it
                comp.wait_event(self.fetched[slot])
            with torch.cuda.stream(comp):
                if self.split[slot] is not None:
                    self.split[slot][0].replay()
                    self.read[slot].record(comp)
                    self.split[slot][1].replay()
                else:
                    self.graphs[slot].replay()
                rec = pack(self.engines[slot].topk()) if pack is not None else self.slots[slot][2]
                self.done[slot].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.done[slot])
                host_out[i].copy_(rec, non_blocking=True)
                rec.record_stream(self.d2h)
                self.fetched[slot].record(self.d2h)
        for c in comps:
            if c is not main:
                main.wait_stream(c)
        main.wait_stream(self.d2h)
