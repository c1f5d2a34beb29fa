"""Per-role timeline of one tcgen05 conv launch (CTA 0): prologue, producer / MMA /
epilogue hand-offs per tile, teardown -- plus the launch's event-timed duration.

    python tools/conv_trace.py [int8|fp16] [batch] [h w cin cout stride]
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12638_b200 import _native as N  # noqa: E402


def main():
    lib = N.load()
    prec = sys.argv[1] if len(sys.argv) > 1 else "int8"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    h, w, cin, cout, st = (int(v) for v in sys.argv[3:8]) if len(sys.argv) > 7 else (248, 216, 64, 64, 1)
    oh, ow = (h - 1) // st + 1, (w - 1) // st + 1
    tdt = torch.int8 if prec == "int8" else torch.float16
    x = torch.zeros((B, h, w, cin), dtype=tdt, device="cuda")
    wt = torch.zeros((cout, 9 * cin), dtype=tdt, device="cuda")
    alpha = torch.full((cout,), 1e-3, device="cuda")
    bias = torch.zeros((cout,), device="cuda")
    y = torch.empty((B, oh, ow, cout), dtype=torch.int8, device="cuda")
    desc = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.DTYPE_CODE[prec], batch=B, in_h=h, in_w=w, in_c=cin,
                      in_c_stride=cin, in_c_offset=0, out_c=cout, k_h=3, k_w=3, stride_h=st, stride_w=st, pad_h=1,
                      pad_w=1, out_h=oh, out_w=ow, relu=1)
    arr, n = N.outs_array([N.Out(ptr=y.data_ptr(), scale=0.05, dtype=N.PMX_I8, c_stride=cout, c_offset=0)])
    tr = torch.zeros(10 * 64, dtype=torch.int64, device="cuda")

    def call():
        N.check(lib.pmx_conv(ctypes.byref(desc), x.data_ptr(), wt.data_ptr(), alpha.data_ptr(), bias.data_ptr(),
                             None, arr, n, None, None, 0, N.stream_ptr()))

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        call()
    b.record()
    torch.cuda.synchronize()
    print(f"{prec} B={B} {h}x{w}x{cin}->{cout} s{st}: {1e3 * a.elapsed_time(b) / 50:.1f} us/launch (stream, eager)")
    lib.pmx_debug_trace(tr.data_ptr())
    call()
    torch.cuda.synchronize()
    lib.pmx_debug_trace(None)
    t = tr.cpu().numpy().reshape(10, 64).astype(np.int64)
    t0 = t[8, 0]
    print("prologue: setup %d, weights landed %d, teardown %d (cycles from entry)" %
          tuple((t[8, i] - t0) if t[8, i] else -1 for i in (1, 2, 3)))
    names = ["P.wait_empty", "P.issued", "M.wait_full", "M.full_ok", "M.committed", "E.wait_tfull", "E.tfull_ok",
             "E.released", "", "M.loop_top"]
    print("tile " + " ".join(f"{names[e]:>12}" for e in (0, 1, 9, 2, 3, 4, 5, 6, 7)))
    for i in range(24):
        if not t[:8, i].any() and not t[9, i]:
            break
        print(f"{i:4d} " + " ".join(f"{(t[e, i] - t0) if t[e, i] else -1:12d}" for e in (0, 1, 9, 2, 3, 4, 5, 6, 7)))


if __name__ == "__main__":
    main()
