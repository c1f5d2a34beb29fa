"""Per-role timeline of one tcgen05 conv launch (CTA 0): producer / MMA / epilogue hand-offs."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12638_b200 import _native as N  # noqa: E402


def main():
    lib = N.load()
    B, h, w, cin, cout = 32, 248, 216, 64, 64
    prec = sys.argv[1] if len(sys.argv) > 1 else "int8"
    mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    tdt = torch.int8 if prec == "int8" else torch.float16
    x = torch.zeros((B, h, w, cin), dtype=tdt, device="cuda")
    wt = torch.zeros((cout, 9 * cin), dtype=tdt, device="cuda")
    alpha = torch.full((cout,), 1e-3, device="cuda")
    bias = torch.zeros((cout,), device="cuda")
    y = torch.empty((B, h, w, cout), dtype=torch.int8, device="cuda")
    desc = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.DTYPE_CODE[prec], batch=B, in_h=h, in_w=w, in_c=cin,
                      in_c_stride=cin, in_c_offset=0, out_c=cout, k_h=3, k_w=3, stride_h=1, stride_w=1, pad_h=1,
                      pad_w=1, out_h=h, out_w=w, relu=1)
    arr, n = N.outs_array([N.Out(ptr=y.data_ptr(), scale=0.05, dtype=N.PMX_I8, c_stride=cout, c_offset=0)])
    tr = torch.zeros(8 * 64, dtype=torch.int64, device="cuda")
    lib.pmx_set_conv_backend(mode)
    for k in range(3):
        if k == 2:
            lib.pmx_debug_trace(tr.data_ptr())
        N.check(lib.pmx_conv(ctypes.byref(desc), x.data_ptr(), wt.data_ptr(), alpha.data_ptr(), bias.data_ptr(), None,
                             arr, n, None, None, 0, N.stream_ptr()))
        torch.cuda.synchronize()
    lib.pmx_debug_trace(None)
    t = tr.cpu().numpy().reshape(8, 64).astype(np.int64)
    t0 = t[t > 0].min()
    names = ["P.wait_empty", "P.issued", "M.wait_full", "M.full_ok", "M.committed", "E.wait_tfull", "E.tfull_ok",
             "E.released"]
    print("tile " + " ".join(f"{n:>12}" for n in names))
    for i in range(24):
        print(f"{i:4d} " + " ".join(f"{(t[e, i] - t0) if t[e, i] else -1:12d}" for e in range(8)))


if __name__ == "__main__":
    main()
