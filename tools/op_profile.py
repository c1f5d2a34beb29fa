"""Run ONE engine op of the real pipeline (real activations) inside a profiler range,
for `ncu --profile-from-start off` captures:

    ncu --set full --profile-from-start off -o gpurun_out/x python tools/op_profile.py \
        --op "conv backbone.blocks.0.3" [--batch 32] [--plan "FP16: 2,18,19,20"]
    python tools/op_profile.py --list
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_12638_b200 as pm  # noqa: E402
from paper_2601_12638_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="conv backbone.blocks.0.3", help='an op name (--list) or "all"')
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--points", type=int, default=120000)
    ap.add_argument("--plan", default="FP16: 2,18,19,20")
    ap.add_argument("--list", action="store_true")
    ap.add_argument("--trace", action="store_true", help="print CTA 0's per-tile timeline (tcgen05 convs)")
    ap.add_argument("--time", action="store_true", help="CUDA-event time of the op (eager, 20 reps)")
    args = ap.parse_args()
    cfg = pm.PointPillarsConfig(max_pillars=16000)
    graph = pm.build_pointpillars(cfg, seed=0)
    stats = pm.calibrate_frames(graph, [pm.make_frame(args.points, 900 + i, cfg, 0.01) for i in range(2)], cfg)
    eng = pm.PointPillarsEngine(graph, args.plan, stats, cfg, batch=args.batch, max_points_per_frame=args.points)
    eng.load_points([pm.make_frame(args.points, 5 + i, cfg) for i in range(args.batch)])
    if args.list:
        print("\n".join(name for name, _ in eng.cg.ops))
        return
    for _ in range(2):
        eng.run()
    torch.cuda.synchronize()
    if args.op == "all":  # one whole eager step (every op in order) inside the profiler range
        def fn(stream):
            for _, f in eng.cg.ops:
                f(stream)
    else:
        fn = dict(eng.cg.ops)[args.op]
    if args.time:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            fn(N.stream_ptr())
        b.record()
        torch.cuda.synchronize()
        print(f"{args.op}: {1e3 * a.elapsed_time(b) / 20:.1f} us")
    if args.trace:
        import numpy as np

        lib = N.load()
        tr = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
        lib.pmx_debug_trace(tr.data_ptr())
        fn(N.stream_ptr())
        torch.cuda.synchronize()
        lib.pmx_debug_trace(None)
        t = tr.cpu().numpy().reshape(16, 64).astype(np.int64)
        t0 = t[8, 0]
        print("prologue: setup %d, weights landed %d, teardown %d (cycles from entry)" %
              tuple((t[8, i] - t0) if t[8, i] else -1 for i in (1, 2, 3)))
        names = ["P.wait_empty", "P.issued", "M.wait_full", "M.full_ok", "M.committed", "E.wait_tfull",
                 "E.tfull_ok", "E.released", "", "M.loop_top"]
        print("tile " + " ".join(f"{names[e]:>12}" for e in (0, 1, 9, 2, 3, 4, 5, 6, 7)))
        print("tile 6 per epilogue warp (tfull_ok, released): " +
              " ".join(f"w{w + 2}:{t[8, 8 + 2 * w] - t0}/{t[8, 9 + 2 * w] - t0}" for w in range(16)))
        for i in range(32):
            if not t[:8, i].any() and not t[9, i]:
                break
            print(f"{i:4d} " + " ".join(f"{(t[e, i] - t0) if t[e, i] else -1:12d}" for e in (0, 1, 9, 2, 3, 4, 5, 6, 7)))
        if t[10].any():
            print("gather producer (thread 0): iter_start, empty_ok, arrived")
            for i in range(32):
                print(f"{i:4d} " + " ".join(f"{(t[e, i] - t0) if t[e, i] else -1:10d}" for e in (0, 10, 1)))
        return
    torch.cuda.profiler.start()
    fn(N.stream_ptr())
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
