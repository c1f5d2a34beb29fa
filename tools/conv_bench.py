"""Per-layer timing of pmx_conv at the PointPillars shapes (CUDA events, no profiler).
    python tools/conv_bench.py [--batch 32] [--prec int8|fp16] [--simt]"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12638_b200 import _native as N  # noqa: E402

LAYERS = [  # name, kind, cin, cout, k, s, in (h, w)
    ("blocks.0.0", "conv", 64, 64, 3, 2, (496, 432)),
    ("blocks.0.x", "conv", 64, 64, 3, 1, (248, 216)),
    ("blocks.1.0", "conv", 64, 128, 3, 2, (248, 216)),
    ("blocks.1.x", "conv", 128, 128, 3, 1, (124, 108)),
    ("blocks.2.0", "conv", 128, 256, 3, 2, (124, 108)),
    ("blocks.2.x", "conv", 256, 256, 3, 1, (62, 54)),
    ("deblock.0", "deconv", 64, 128, 1, 1, (248, 216)),
    ("deblock.1", "deconv", 128, 128, 2, 2, (124, 108)),
    ("deblock.2", "deconv", 256, 128, 4, 4, (62, 54)),
    ("heads", "conv", 384, 20, 1, 1, (248, 216)),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--prec", default="int8")
    ap.add_argument("--simt", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    lib = N.load()
    lib.pmx_set_conv_backend(1 if args.simt else 0)
    B = args.batch
    res = []
    for name, kind, cin, cout, k, s, (h, w) in LAYERS:
        deconv = kind == "deconv"
        if deconv:
            oh, ow, ng, K = h * s, w * s, k * k * cout, cin
        else:
            pad = 1 if k == 3 else 0
            oh, ow, ng, K = (h + 2 * pad - k) // s + 1, (w + 2 * pad - k) // s + 1, cout, k * k * cin
        dt = N.DTYPE_CODE[args.prec]
        tdt = {"int8": torch.int8, "fp16": torch.float16, "fp32": torch.float32}[args.prec]
        x = torch.zeros((B, h, w, cin), dtype=tdt, device="cuda")
        wt = torch.zeros((ng, K), dtype=tdt, device="cuda")
        alpha = torch.full((cout,), 1e-3, device="cuda")
        bias = torch.zeros((cout,), device="cuda")
        out_dt = N.PMX_I8 if name != "heads" else N.PMX_F32
        y = torch.empty((B, oh, ow, cout), dtype=torch.int8 if out_dt == N.PMX_I8 else torch.float32, device="cuda")
        desc = N.ConvDesc(kind=N.PMX_DECONV2D if deconv else N.PMX_CONV2D, in_dtype=dt, batch=B, in_h=h, in_w=w,
                          in_c=cin, in_c_stride=cin, in_c_offset=0, out_c=cout, k_h=k, k_w=k, stride_h=s, stride_w=s,
                          pad_h=0 if deconv or k == 1 else 1, pad_w=0 if deconv or k == 1 else 1, out_h=oh, out_w=ow,
                          relu=1)
        arr, n = N.outs_array([N.Out(ptr=y.data_ptr(), scale=0.05, dtype=out_dt, c_stride=cout, c_offset=0)])

        def run():
            N.check(lib.pmx_conv(ctypes.byref(desc), x.data_ptr(), wt.data_ptr(), alpha.data_ptr(), bias.data_ptr(),
                                 None, arr, n, None, None, 0, N.stream_ptr()), name)

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.reps
        flops = 2.0 * B * (h * w if deconv else oh * ow) * ng * K
        esz = {"int8": 1, "fp16": 2, "fp32": 4}[args.prec]
        bytes_ = B * h * w * cin * esz + ng * K * esz + B * oh * ow * cout * (1 if out_dt == N.PMX_I8 else 4)
        res.append({"layer": name, "us": round(ms * 1e3, 1), "TFLOPs": round(flops / ms / 1e9, 1),
                    "GBs": round(bytes_ / ms / 1e6, 1), "backend": lib.pmx_conv_backend(dt, desc.kind).decode()})
        print(json.dumps(res[-1]), flush=True)
    lib.pmx_set_conv_backend(0)


if __name__ == "__main__":
    main()
