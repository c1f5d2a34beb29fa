import ctypes, os
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "store_probe.so"))
lib.probe.restype = ctypes.c_float
MB = 53568 * 32 * 128 / 1e6
for kind in (0, 1, 2):
    for s16 in (8, 16, 24):
        us = lib.probe(kind, s16, 20)
        print(f"{['coalesced', 'per_pixel', 'seg64'][kind]:10s} row stride {s16 * 16:4d} B: {us:8.1f} us  {MB / us * 1e3 / 1e3:7.2f} TB/s written")
