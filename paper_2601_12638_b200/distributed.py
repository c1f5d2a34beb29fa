"""Multi-GPU plumbing: one process per GPU, frames (or sweep plans) sharded by rank.

The per-frame path has no exchange step: each rank runs the whole
engine on its own frames.  NCCL (``torch.distributed``) appears only after a
batch -- to gather fixed-size per-frame top-k records and per-rank timings --
and after a sweep phase -- to gather per-plan error sums.  The same functions
run on ``gloo`` for the CPU tests.
"""

from __future__ import annotations

import os

import numpy as np

__all__ = ["init_from_env", "free_port", "spawn_ranks", "shard_range", "shard_round_robin", "pack_topk", "gather_records", "max_over_ranks",
           "gather_scalars"]

RECORD = 10  # per detection: idx, logit, x, y, z, w, l, h, yaw, dir


def init_from_env(backend: str | None = None):
    """torchrun-style env (RANK, WORLD_SIZE, LOCAL_RANK, MASTER_ADDR/PORT) -> (rank, world, local_rank)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world, local


def free_port() -> int:
    """An unused TCP port on 127.0.0.1 (rendezvous for spawned ranks)."""
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(script: str, n: int, argv: list[str]) -> int:
    """Re-run ``script argv`` as ``n`` ranks under torch.distributed.run (one process per
    GPU, rendezvous on 127.0.0.1 at a free port) and return the launcher's exit code.
    Used when a multi-GPU run is requested without an outer torchrun."""
    import subprocess
    import sys

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *argv]
    return subprocess.call(cmd)


def shard_range(n_items: int, rank: int, world: int) -> range:
    """Contiguous block of items for this rank (frames: rank r takes [r*B, (r+1)*B))."""
    per = (n_items + world - 1) // world
    return range(min(rank * per, n_items), min((rank + 1) * per, n_items))


def shard_round_robin(items, rank: int, world: int):
    """Round-robin shard (sweep plans: independent candidates)."""
    return [it for i, it in enumerate(items) if i % world == rank]


def pack_topk(topk: dict):
    """Engine top-k dict -> fixed-size float32 records [B, k, 10] (idx < 2^24 is exact in f32)."""
    import torch

    idx = topk["idx"].to(torch.float32).unsqueeze(-1)
    logit = topk["logit"].unsqueeze(-1)
    dr = topk["dir"].to(torch.float32).unsqueeze(-1)
    return torch.cat([idx, logit, topk["boxes"], dr], dim=-1).contiguous()


def gather_records(records, group=None):
    """all_gather_into_tensor of equal-size per-rank records -> [world * B, k, R] on every rank."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return records
    world = dist.get_world_size(group)
    out = torch.empty((world * records.shape[0],) + tuple(records.shape[1:]), dtype=records.dtype,
                      device=records.device)
    dist.all_gather_into_tensor(out, records.contiguous(), group=group)
    return out


def gather_scalars(values, device=None, group=None) -> np.ndarray:
    """Per-rank f64 vectors (e.g. per-plan sum of squared errors) -> [world, n] on every rank."""
    import torch

    t = torch.as_tensor(np.asarray(values, np.float64), device=device)
    return gather_records(t.reshape(1, -1), group).cpu().numpy()


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (step time) over ranks."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
