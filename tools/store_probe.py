"""Store-pattern probe: write a [M,128] int8 block into (a) a dense [M,128] buffer,
(b) the first 128 channels of a [M,384] concat buffer, (c) other slices, via torch copies."""
import torch

M = 53568 * 32
src = torch.randint(-128, 127, (M, 128), dtype=torch.int8, device="cuda")
dense = torch.empty((M, 128), dtype=torch.int8, device="cuda")
cat = torch.empty((M, 384), dtype=torch.int8, device="cuda")
cat2 = torch.empty((M, 256), dtype=torch.int8, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for name, fn in [("dense", lambda: dense.copy_(src)), ("cat384[:, :128]", lambda: cat[:, :128].copy_(src)),
                 ("cat384[:, 256:]", lambda: cat[:, 256:].copy_(src)), ("cat256[:, :128]", lambda: cat2[:, :128].copy_(src)),
                 ("cat384 full", lambda: cat.copy_(torch.cat([src, src, src], 1)) if False else cat.fill_(1))]:
    us = t(fn)
    print(f"{name:20s} {us:8.1f} us  {2 * M * 128 / us / 1e3:7.1f} GB/s (r+w of 128 B/row)")
