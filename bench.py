"""Benchmark: mixed INT8/FP16 PointPillars frames/s (config 4) + batch-1 p50 latency vs FP32.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path (GPU pillarize -> PFN+scatter -> 16 convs ->
3 deconvs -> 3 heads -> anchor top-k) over a batch of B=32 synthetic KITTI-shaped
frames per GPU with 60k-150k points each (seeded; BASELINE config 4), plan
"FP16: 2,18,19,20" (config 3), PTQ stats from 2 calibration frames.  The step is
replayed from one CUDA graph.  Multi-GPU: torchrun, one process per GPU, frames
sharded by rank (weak scaling), time = max over ranks, NCCL only gathers the
per-frame top-k records after the timed region.  Prints one JSON line on rank 0.
"""

from __future__ import annotations

import os
import sys

NCORES = len(os.sched_getaffinity(0))
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(NCORES))  # before numpy loads

import argparse  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "mixed INT8/FP16 PointPillars frames/s and p50 batch-1 latency ms vs FP32"
BATCH = 32
N_RANGE = (60000, 150000)
MAX_PILLARS = 16000
CALIB_FRAMES = 2


def _mma_peaks(peaks):
    """Dense tcgen05 MMA peaks per layer dtype (TFLOP/s): the measured probe when committed,
    else the bf16 cuBLAS number of MEASURED_PEAKS.json (fp16) and twice that (int8)."""
    f = ROOT / "profiles" / "r2_mma_peak.json"
    if f.exists():
        d = json.loads(f.read_text())
        return ({"int8": d["int8_tops_burst"], "fp16": d["f16_tflops_burst"], "fp32x2": d["tf32_tflops_burst"] / 3.0},
                "measured tcgen05 MMA burst peaks (profiles/r2_mma_peak.json, tools/mma_peak.cu): FLOP-weighted "
                "mix of the int8 and f16 peaks over the layers")
    return ({"fp16": peaks["bf16_tflops"], "int8": 2.0 * peaks["bf16_tflops"]},
            "MEASURED_PEAKS.json bf16 burst (fp16 layers) and 2x bf16 (int8 layers)")


def torch_dist_done():
    import torch.distributed as dist

    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons = [], 0.0, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_frame(pm, O, graph, stats, cfg, frame, plan):
    """The CPU path on one frame: oracle pillarize + planned forward (numpy/OpenBLAS) + top-k decode."""
    planned = pm.apply_plan(pm.fold_all_bn(graph), plan)
    precs = {l.index: l.precision.value for l in planned.weight_layers}
    sample, _ = O.pillarize_kitti(frame, cfg.grid_spec())
    heads = O.forward(O.folded_graph(planned, precs), sample, stats=stats)
    O.topk_anchor_order(heads[2][0], cfg.topk)
    return heads


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port of pillarmix) on host cores."""
    if rank != 0:
        return
    import paper_2601_12638_b200 as pm
    from oracle import pillars_oracle as O

    cfg = pm.PointPillarsConfig(max_pillars=MAX_PILLARS)
    graph = pm.build_pointpillars(cfg, seed=0)
    plan = pm.parse_plan_label(pm.MIXED_PLAN_LABEL)
    calib = [pm.make_frame(120000, 900 + i, cfg, outlier_frac=0.01) for i in range(CALIB_FRAMES)]
    ranges = O.per_sample_ranges(graph, [O.pillarize_kitti(f, cfg.grid_spec())[0] for f in calib])
    stats = pm.calibration.stats_from_ranges(graph, ranges, per_channel_weights=True)
    frames = pm.make_frames(args.warmup + args.steps, 1000, cfg, N_RANGE)
    for f in frames[: args.warmup]:
        cpu_reference_frame(pm, O, graph, stats, cfg, f, plan)
    t0 = time.perf_counter()
    for f in frames[args.warmup:]:
        cpu_reference_frame(pm, O, graph, stats, cfg, f, plan)
    dt = time.perf_counter() - t0
    fps = args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8/fp16 (fake-quant f32 numpy)", "data": "synthetic",
        "config": {"workload": "C4 frames (60k-150k pts), mixed plan " + pm.MIXED_PLAN_LABEL + ", 1 frame per step",
                   "plan": pm.MIXED_PLAN_LABEL, "max_pillars": MAX_PILLARS},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": NCORES, "kind": "port",
                         "sample": f"{args.steps} frames of config 4, 1 frame per step, OPENBLAS_NUM_THREADS={NCORES}"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def launch_check(args, D):
    """Every rank joins the process group (NCCL with GPUs, gloo without), the ranks agree
    on the world size and the max over ranks; rank 0 prints one JSON line."""
    import torch

    backend = "nccl" if torch.cuda.is_available() else "gloo"
    rank, world, local = D.init_from_env(backend)
    dev = None
    if backend == "nccl":
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    mx = D.max_over_ranks(float(rank), device=dev)
    ranks = D.gather_scalars([rank], device=dev).ravel().astype(int).tolist()
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "backend": backend, "max_rank": mx,
                          "ranks": ranks}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def b1_latency(pm, graph, stats, cfg, plan, n_points, seed, reps=200):
    import torch

    frame = pm.make_frame(n_points, seed, cfg)
    e = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=1, max_points_per_frame=n_points)
    e.load_points([frame])
    e.capture()
    for _ in range(10):
        e.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        e.run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.percentile(ts, 50)), float(np.percentile(ts, 99))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--inflight", type=int, default=2, choices=[1, 2],
                    help="captured step instances in flight (own buffers, one stream each)")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launch-check", action="store_true",
                    help="only start the ranks, agree on the world size and exit (tests the multi-rank launch)")
    args = ap.parse_args()

    from paper_2601_12638_b200 import distributed as D

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no outer torchrun: start one rank per GPU ourselves (127.0.0.1, free port)
        sys.exit(D.spawn_ranks(str(Path(__file__).resolve()), args.gpus, sys.argv[1:]))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env} ranks were launched")
    if args.launch_check:
        launch_check(args, D)
        return
    rank, world, local = D.init_from_env("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            torch_dist_done()
        return
    import torch

    import paper_2601_12638_b200 as pm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    args.warmup = max(args.warmup, 3)
    cfg = pm.PointPillarsConfig(max_pillars=MAX_PILLARS)
    graph = pm.build_pointpillars(cfg, seed=0)
    plan = pm.parse_plan_label(pm.MIXED_PLAN_LABEL)
    calib = [pm.make_frame(120000, 900 + i, cfg, outlier_frac=0.01) for i in range(CALIB_FRAMES)]
    stats = pm.calibrate_frames(graph, calib, cfg, per_channel_weights=True)
    B = args.batch
    frames = pm.make_frames(B, 1000 + rank, cfg, N_RANGE)
    eng = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=B, max_points_per_frame=N_RANGE[1])
    eng.load_points(frames)

    # per-op device times (each op replayed from its own CUDA graph between CUDA events
    # on the launching stream) -> dominant kernel roofline
    op_ms = eng.cg.timed_ops(reps=10)
    eng.capture()
    # a second captured instance (own activation buffers) keeps two batches in flight on
    # two streams: one batch's kernel tails and launch gaps are filled by the other's
    # kernels (tools/multistream_probe.py: 1 / 2 / 3 instances measured; 2 is best)
    engines = [eng]
    if args.inflight > 1:
        eng2 = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=B, max_points_per_frame=N_RANGE[1])
        eng2.load_points(frames)
        eng2.capture()
        engines.append(eng2)
    streams = [torch.cuda.Stream() for _ in engines]

    def run_steps(n):
        t0 = torch.cuda.Event()
        t0.record()
        for st in streams:
            st.wait_event(t0)
        for i in range(n):
            with torch.cuda.stream(streams[i % len(engines)]):
                engines[i % len(engines)].run()
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)

    run_steps(args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    run_steps(args.steps)
    end.record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    ms_local = start.elapsed_time(end) / args.steps
    ms = D.max_over_ranks(ms_local, device=dev)
    value = B * world / (ms / 1e3)

    # e2e through the public API with host buffers: pinned points H2D + graph + top-k D2H, every step
    host_pts = torch.from_numpy(np.concatenate(frames)).pin_memory()
    offs = np.zeros(B + 1, np.int64)
    offs[1:] = np.cumsum([len(f) for f in frames])
    host_offs = torch.from_numpy(offs).pin_memory()
    rec_dev = D.pack_topk(eng.topk())
    h2d = host_pts.numel() * 4 + host_offs.numel() * 8
    d2h = rec_dev.numel() * 4

    # the public streaming API: batch i+1's H2D (pinned host -> device) overlaps batch
    # i's graph, batch i's records come back D2H; every step pays its own copies
    pipe = pm.PipelinedEngine(eng, engines[1] if len(engines) > 1 else None)
    host_recs = [torch.empty(rec_dev.shape, dtype=rec_dev.dtype).pin_memory() for _ in range(2)]
    pipe.run([(host_pts, host_offs)] * args.warmup, [host_recs[i % 2] for i in range(args.warmup)])
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    start.record()
    pipe.run([(host_pts, host_offs)] * args.steps, [host_recs[i % 2] for i in range(args.steps)])
    end.record()
    torch.cuda.synchronize()
    e2e_ms = D.max_over_ranks(start.elapsed_time(end) / args.steps, device=dev)
    e2e_value = B * world / (e2e_ms / 1e3)

    # NCCL: gather per-rank top-k records (outside the per-frame path)
    gathered = D.gather_records(D.pack_topk(eng.topk()))

    # roofline for the dominant kernel class
    peaks, peak_src = _peaks()
    info = eng.cg.op_info
    conv_ms = sum(v for k, v in op_ms.items() if k.startswith("conv "))
    conv_flops = sum(info[k]["flops"] for k in info)
    by_class = {}
    for k, v in op_ms.items():
        by_class[k.split(" ")[0]] = by_class.get(k.split(" ")[0], 0.0) + v
    dominant = max(by_class, key=by_class.get)
    step_ms_eager = sum(op_ms.values())
    if dominant == "conv":
        # tensor roofline of the layer mix: each layer at its own dtype's dense tcgen05 peak,
        # measured on this pool by tools/mma_peak.cu (profiles/r2_mma_peak.json: back-to-back
        # M=128 N=256 MMAs on every SM, burst -- every op is timed alone from its own graph)
        pk, pk_src = _mma_peaks(peaks)
        t_min = sum(info[k]["flops"] / (pk.get(info[k]["precision"], peaks["bf16_tflops"]) * 1e12) for k in info)
        peak = conv_flops / t_min / 1e12
        t_bound = sum(max(info[k]["flops"] / (pk.get(info[k]["precision"], peaks["bf16_tflops"]) * 1e12),
                          info[k].get("bytes", 0) / (peaks["hbm_gbs"] * 1e9)) for k in info)
        achieved = conv_flops / (conv_ms / 1e3) / 1e12
        # DRAM traffic of the same 20 conv launches (one step, batch 32) from the committed ncu
        # capture (tools/traffic.py) next to their algorithmic bytes
        traffic = None
        tf = ROOT / "profiles" / "r2_step_traffic.json"
        if not tf.exists():
            tf = ROOT / "profiles" / "r1_step_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get("conv_dram_bytes")
        alg_bytes = sum(info[k].get("bytes", 0) for k in info)
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "traffic_note": f"bytes per step: DRAM read+write of the conv launches (ncu, "
                                    f"profiles/{tf.name}) vs algorithmic_bytes (each layer's input + "
                                    "weights + outputs once)",
                    "algorithmic_bytes": alg_bytes,
                    "kernel": "pmx_conv implicit GEMM, all 20 conv/deconv/head launches of a step",
                    "algorithmic": f"{conv_flops / B / 1e9:.2f} GFLOP/frame x {B} frames per step",
                    "share_of_step": conv_ms / step_ms_eager,
                    "peak_source": pk_src,
                    "peaks_tflops": pk,
                    "per_layer_ms": {k: round(op_ms[k], 4) for k in info},
                    "per_layer": {k: {"ms": round(op_ms[k], 5), "flops": info[k]["flops"],
                                      "bytes": info[k].get("bytes", 0), "precision": info[k]["precision"]}
                                  for k in info},
                    # per-layer max(FLOP / dtype peak, algorithmic bytes / HBM): the bound with the
                    # memory-bound layers (deconvs, heads, stride-2 convs) counted as such
                    "layer_bound_ms": round(t_bound * 1e3, 4), "frac_of_layer_bound": t_bound * 1e3 / conv_ms,
                    "backend": pm._native.load().pmx_conv_backend(2, 0).decode()}
    else:
        roofline = {"bound": "hbm", "achieved": None, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": None,
                    "traffic": None, "kernel": dominant, "share_of_step": by_class[dominant] / step_ms_eager}

    lat = None
    if not args.no_latency:
        # config 3 (mixed, 120k points) and config 1 (FP32, 20k points / 12000 pillars) at batch 1,
        # plus FP32 on the config-3 frame itself (same geometry both sides) and config 2
        # (all-INT8, per-channel weights, 4 calibration frames with 1% outliers)
        mixed_p50, mixed_p99 = b1_latency(pm, graph, stats, cfg, plan, 120000, 77)
        fp32_c3_p50, _ = b1_latency(pm, graph, None, cfg, pm.PrecisionPlan(), 120000, 77)
        cfg1 = pm.PointPillarsConfig(max_pillars=12000)
        fp32_p50, fp32_p99 = b1_latency(pm, graph, None, cfg1, pm.PrecisionPlan(), 20000, 78)
        calib4 = [pm.make_frame(120000, 900 + i, cfg, outlier_frac=0.01) for i in range(4)]
        stats_c2 = pm.calibrate_frames(graph, calib4, cfg, per_channel_weights=True)
        int8_p50, int8_p99 = b1_latency(pm, graph, stats_c2, cfg, pm.parse_plan_label("INT8"), 120000, 77)
        # config 3 batch-8 throughput (the same captured step as the headline, 8 frames)
        f8 = pm.make_frames(8, 3000, cfg, (120000, 120000))
        e8 = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=8, max_points_per_frame=120000)
        e8.load_points(f8)
        e8.capture()
        for _ in range(5):
            e8.run()
        a8, b8 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a8.record()
        for _ in range(50):
            e8.run()
        b8.record()
        torch.cuda.synchronize()
        ms8 = a8.elapsed_time(b8) / 50
        del e8
        lat = {"mixed_b1_p50_ms": mixed_p50, "mixed_b1_p99_ms": mixed_p99, "fp32_b1_p50_ms": fp32_p50,
               "fp32_b1_p99_ms": fp32_p99, "fp32_over_mixed": fp32_p50 / mixed_p50,
               "mixed_shape": "C3: 120k pts, 16000 pillars", "fp32_shape": "C1: 20k pts, 12000 pillars",
               "fp32_c3_b1_p50_ms": fp32_c3_p50, "fp32_over_mixed_same_frame": fp32_c3_p50 / mixed_p50,
               "int8_c2_b1_p50_ms": int8_p50, "int8_c2_b1_p99_ms": int8_p99,
               "mixed_c3_b8_ms_per_step": ms8, "mixed_c3_b8_frames_per_s": 8 / (ms8 / 1e3),
               "fp32_backend": "3xTF32 tcgen05 (kind::tf32, hi/lo split, f32 accumulate)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import pillars_oracle as O

        t0 = time.perf_counter()
        cpu_reference_frame(pm, O, graph, stats, cfg, frames[0], plan)
        dt = time.perf_counter() - t0
        t0 = time.perf_counter()
        cpu_reference_frame(pm, O, graph, None, cfg, frames[0], pm.PrecisionPlan())
        dt32 = time.perf_counter() - t0
        cpu = {"value": 1.0 / dt, "unit": "frames/s", "cores": NCORES, "kind": "port",
               "sample": f"1 frame ({len(frames[0])} pts) of the config-4 batch: oracle pillarize + mixed-plan "
                         f"forward (numpy/OpenBLAS, {NCORES} threads) + top-k",
               "fp32_value": 1.0 / dt32, "fp32_sample": "the same frame, FP32 plan"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int8/fp16 (plan " + pm.MIXED_PLAN_LABEL + "), int32/f32 accumulate",
            "data": "synthetic (seeded KITTI-shaped frames, random-init weights)",
            "config": {"workload": "C4: mixed plan, batch 32 frames/GPU, 60k-150k points/frame",
                       "plan": pm.MIXED_PLAN_LABEL, "global_batch": B * world, "max_pillars": MAX_PILLARS,
                       "parallelism": f"frames sharded over {world} GPU(s)",
                       "l2": "inputs larger than L2 (per-step activations > 1 GB)", "calib_frames": CALIB_FRAMES,
                       "in_flight": f"{len(engines)} captured instances of the step (own buffers), steps "
                                    f"alternating over {len(engines)} streams"},
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "gpu_launches": eng.cg.kernels_per_launch() * args.steps,
            "clocks": clk,
            "latency": lat,
            "op_ms": {k: round(v, 4) for k, v in by_class.items()},
            "gathered_records": list(gathered.shape),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
