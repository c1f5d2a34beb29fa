"""N>1 host logic on CPU: world_size-2 gloo process group, frame sharding, top-k record
gather and max-over-ranks timing (the NCCL calls bench.py makes on the GPU box)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2601_12638_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r, w, _ = D.init_from_env("gloo")
    frames = list(D.shard_range(2 * 32, r, w))
    k = 5
    topk = {"idx": torch.arange(len(frames) * k, dtype=torch.int32).reshape(len(frames), k) + 1000 * r,
            "logit": torch.full((len(frames), k), float(r)), "boxes": torch.zeros((len(frames), k, 7)),
            "dir": torch.ones((len(frames), k), dtype=torch.int32)}
    rec = D.gather_records(D.pack_topk(topk))
    t = D.max_over_ranks(1.5 + r)
    sc = D.gather_scalars([r, 2.0 * r])
    plans = D.shard_round_robin(list(range(7)), r, w)
    q.put((r, frames[0], frames[-1], rec.shape, float(rec[32, 0, 0]), float(rec[0, 0, 1]), t, sc.tolist(), plans))
    torch.distributed.destroy_process_group()


def test_two_rank_gather_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, b0, shape0, idx_r1, logit_r0, t0, sc0, pl0), (r1, a1, b1, shape1, _, _, t1, sc1, pl1) = res
    assert (a0, b0, a1, b1) == (0, 31, 32, 63)
    assert tuple(shape0) == (64, 5, D.RECORD) == tuple(shape1)
    assert idx_r1 == 1000.0 and logit_r0 == 0.0
    assert t0 == t1 == 2.5
    assert sc0 == sc1 == [[0.0, 0.0], [1.0, 2.0]]
    assert pl0 == [0, 2, 4, 6] and pl1 == [1, 3, 5]


def _sweep_worker(rank, world, port, q):
    from paper_2601_12638_b200.sweep import sharded_plan_sums

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r, w, _ = D.init_from_env("gloo")
    seen = []

    def run_plans(js):  # plan j -> (err, ref) = (j + 1, 10 * (j + 1)); records which rank ran it
        seen.extend(js)
        return np.array([[j + 1.0, 10.0 * (j + 1)] for j in js])

    tot = sharded_plan_sums(23, r, w, None, run_plans)
    q.put((r, seen, tot.tolist()))
    torch.distributed.destroy_process_group()


def test_two_rank_sweep_sharding():
    """Config-5 sweep plumbing: 23 single-INT8 plans round-robin over 2 ranks, each plan
    run exactly once, the gathered (err, ref) sums identical on both ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, s0, t0), (_, s1, t1) = res
    assert s0 == list(range(0, 23, 2)) and s1 == list(range(1, 23, 2))
    want = [[j + 1.0, 10.0 * (j + 1)] for j in range(23)]
    assert t0 == t1 == want


def test_bench_spawns_ranks_itself():
    """`bench.py --gpus 2` without an outer torchrun launches its own two ranks (torchrun
    re-exec, 127.0.0.1, free port); here they rendezvous over gloo on the CPU."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--launch-check"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["max_rank"] == 1.0 and lines[0]["ranks"] == [0, 1]


def test_bench_rejects_mismatched_world():
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--launch-check"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
