"""Layer-sensitivity sweep and greedy FP16 candidates (BASELINE config 5).

The paper's procedure: quantize one layer at a
time to INT8 on an FP32 base (the other layers untouched), score each candidate,
rank layers most-sensitive first, then build the greedy plans "FP16: r1",
"FP16: r1,r2", ... on an INT8 base.  With random weights there is no AP to score,
so the score is the head-output error against the FP32 engine on the same frames
(BASELINE config 5): rel_err = sqrt(sum (y - y_fp32)^2 / sum y_fp32^2) over all
heads and frames, accumulated in f64 by the deterministic K12 kernel.
Ties rank the lower layer index first.

Multi-GPU: candidate plans are sharded round-robin over ranks
(``distributed.shard_round_robin``); per-plan (err, ref) pairs are all-gathered
(NCCL on the GPU box) -- no collective inside a forward.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .model import PrecisionPlan, parse_plan_label
from .pointpillars import PointPillarsConfig, PointPillarsEngine
from .quant import DType

__all__ = ["SensitivityRecord", "head_error", "plan_errors", "sensitivity_sweep", "select_topk",
           "greedy_candidates", "exhaustive_subsets", "exhaustive_search", "sharded_plan_sums", "records"]

EXHAUSTIVE_GUARD = 10_000  # SPEC.md:395 "guard: <= 10^4" subsets


@dataclass(frozen=True)
class SensitivityRecord:
    layer_index: int
    rel_err: float
    rank: int


def sq_err_workspace(lib):
    import torch

    return torch.empty(lib.pmx_sq_err_workspace() // 8, dtype=torch.float64, device="cuda")


def _sq_err(lib, a, b, acc, ws):
    N.check(lib.pmx_sq_err(a.data_ptr(), b.data_ptr(), a.numel(), acc.data_ptr(), ws.data_ptr(),
                           ws.numel() * ws.element_size(), N.stream_ptr()),
            "sq_err")


def _frame_batches(frames, batch):
    for i in range(0, len(frames), batch):
        chunk = frames[i:i + batch]
        if len(chunk) < batch:  # pad the last batch with repeats; their error is not counted
            chunk = chunk + [chunk[-1]] * (batch - len(chunk))
        yield i, chunk


def reference_heads(graph, frames, cfg: PointPillarsConfig, batch: int):
    """FP32 head blocks of every frame, kept resident on the device: [n_frames, H, W, 10A]."""
    import torch

    nmax = max(len(f) for f in frames)
    eng = PointPillarsEngine(graph, PrecisionPlan(), None, cfg, batch=batch, max_points_per_frame=nmax,
                             decode=True)
    out = []
    for i, chunk in _frame_batches(frames, batch):
        eng.load_points(chunk)
        eng.run()
        n = min(batch, len(frames) - i)
        out.append(eng.cg.heads_cat[:n].clone())
    return torch.cat(out, dim=0)


def plan_errors(graph, stats, frames, plans, ref, cfg: PointPillarsConfig, batch: int):
    """(sum_sq_err, sum_sq_ref) per plan against the resident FP32 heads."""
    import torch

    lib = N.require_cuda()
    nmax = max(len(f) for f in frames)
    ws = sq_err_workspace(lib)
    res = []
    for plan in plans:
        eng = PointPillarsEngine(graph, plan, stats, cfg, batch=batch, max_points_per_frame=nmax)
        eng.capture()
        acc = torch.zeros(2, dtype=torch.float64, device="cuda")
        for i, chunk in _frame_batches(frames, batch):
            eng.load_points(chunk)
            eng.run()
            n = min(batch, len(frames) - i)
            _sq_err(lib, eng.cg.heads_cat[:n].contiguous(), ref[i:i + n].contiguous(), acc, ws)
        res.append(acc.cpu().numpy())
        del eng
    return np.array(res).reshape(-1, 2)


def head_error(pair) -> float:
    e, r = float(pair[0]), float(pair[1])
    return float(np.sqrt(e / r)) if r > 0 else float("inf")


def select_topk(errors: dict[int, float], k: int) -> list[int]:
    """Most sensitive first (largest error); ties -> lower layer index."""
    if not 1 <= k <= len(errors):
        raise ValueError(f"k={k} out of range [1, {len(errors)}]")
    return [i for i, _ in sorted(errors.items(), key=lambda kv: (-kv[1], kv[0]))][:k]


def greedy_candidates(ranking: list[int], k: int) -> list[PrecisionPlan]:
    """Candidate i = FP16 on the first i ranked layers, INT8 elsewhere."""
    return [parse_plan_label("FP16: " + ",".join(str(i) for i in ranking[:j])) for j in range(1, k + 1)]


def exhaustive_subsets(layers, k: int, guard: int = EXHAUSTIVE_GUARD) -> list[tuple[int, ...]]:
    """All C(L, k) FP16 subsets in lexicographic index order; refuses
    explicitly, with the count, above the guard."""
    import itertools
    import math

    layers = sorted(layers)
    if not 1 <= k <= len(layers):
        raise ValueError(f"k={k} out of range [1, {len(layers)}]")
    n = math.comb(len(layers), k)
    if n > guard:
        raise ValueError(f"exhaustive search over C({len(layers)}, {k}) = {n} subsets exceeds the guard {guard}")
    return list(itertools.combinations(layers, k))


def exhaustive_search(graph, stats, frames, k: int, cfg: PointPillarsConfig = PointPillarsConfig(),
                      batch: int = 32, layers=None, rank: int = 0, world: int = 1, device=None):
    """The baseline greedy avoids: every k-subset of
    ``layers`` (default: all indexed layers) in FP16 on an INT8 base, scored by the head
    error against FP32 on ``frames``; the best subset has the lowest error, ties to the
    lexicographically first subset.  Plans are sharded round-robin over ranks like the sweep."""
    layers = [l.index for l in graph.weight_layers] if layers is None else list(layers)
    subsets = exhaustive_subsets(layers, k)
    plans = [parse_plan_label("FP16: " + ",".join(str(i) for i in sub)) for sub in subsets]
    ref = reference_heads(graph, frames, cfg, batch)
    tot = sharded_plan_sums(len(plans), rank, world, device,
                            lambda js: plan_errors(graph, stats, frames, [plans[j] for j in js], ref, cfg, batch))
    errs = {sub: head_error(tot[j]) for j, sub in enumerate(subsets)}
    best = min(subsets, key=lambda sub: (errs[sub], sub))
    return {"best": best, "best_error": errs[best], "errors": errs}


def sharded_plan_sums(n_plans: int, rank: int, world: int, device, run_plans) -> np.ndarray:
    """Round-robin the plan indices over ranks, run this rank's share with
    ``run_plans(indices) -> [len, 2]``, all-gather, and return the [n_plans, 2] sums."""
    from . import distributed as D

    mine = D.shard_round_robin(list(range(n_plans)), rank, world)
    local = np.zeros((n_plans, 2))
    if mine:
        local[mine] = run_plans(mine)
    return D.gather_scalars(local.reshape(-1), device=device).reshape(world, n_plans, 2).sum(axis=0)


def sensitivity_sweep(graph, stats, frames, cfg: PointPillarsConfig = PointPillarsConfig(), batch: int = 32,
                      k: int = 5, rank: int = 0, world: int = 1, device=None):
    """Config 5: single-INT8 sweep over every indexed layer + greedy top-1..k FP16 plans.

    Returns a dict with per-layer errors, the ranking, and the candidates' errors;
    every rank returns the same gathered result."""
    ref = reference_heads(graph, frames, cfg, batch)
    layers = [l.index for l in graph.weight_layers]
    singles = [PrecisionPlan(default=DType.FP32, overrides={i: DType.INT8}) for i in layers]
    total = sharded_plan_sums(len(singles), rank, world, device,
                              lambda js: plan_errors(graph, stats, frames, [singles[j] for j in js], ref, cfg, batch))
    errors = {i: head_error(total[j]) for j, i in enumerate(layers)}
    ranking = select_topk(errors, len(errors))
    cands = greedy_candidates(ranking, k)
    ctot = sharded_plan_sums(len(cands), rank, world, device,
                             lambda js: plan_errors(graph, stats, frames, [cands[j] for j in js], ref, cfg, batch))
    return {
        "layer_errors": errors,
        "ranking": ranking,
        "candidates": {c.label(): head_error(ctot[j]) for j, c in enumerate(cands)},
        "n_frames": len(frames),
    }


def records(result) -> list[SensitivityRecord]:
    pos = {i: r for r, i in enumerate(result["ranking"])}
    return [SensitivityRecord(i, e, pos[i] + 1) for i, e in sorted(result["layer_errors"].items())]


def main(argv=None):
    """python -m paper_2601_12638_b200.sweep [--frames 64] [--points 120000] [--k 5]
    (under torchrun for N GPUs: plans sharded round-robin, one JSON line from rank 0)."""
    import argparse
    import json

    import torch

    from . import distributed as D
    from .calibration import calibrate_frames
    from .pointpillars import build_pointpillars, make_frame

    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--points", type=int, default=120000)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--calib", type=int, default=8)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args(argv)
    rank, world, _ = D.init_from_env()
    cfg = PointPillarsConfig()
    graph = build_pointpillars(cfg, seed=args.seed)
    calib = [make_frame(args.points, 7000 + i, cfg, 0.01) for i in range(args.calib)]
    stats = calibrate_frames(graph, calib, cfg)
    frames = [make_frame(args.points, 100 + i, cfg) for i in range(args.frames)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    res = sensitivity_sweep(graph, stats, frames, cfg, batch=min(args.batch, args.frames), k=args.k, rank=rank,
                            world=world, device="cuda")
    t1.record()
    torch.cuda.synchronize()
    dt = D.max_over_ranks(t0.elapsed_time(t1) / 1e3, device="cuda")
    if rank == 0:
        out = {"n_gpus": world, "frames": args.frames, "points": args.points, "seconds": round(dt, 3),
               "plans": len(res["layer_errors"]) + args.k,
               "ranking": res["ranking"],
               "layer_errors": {str(i): e for i, e in res["layer_errors"].items()},
               "candidates": res["candidates"]}
        print(json.dumps(out))
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
