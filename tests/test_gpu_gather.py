"""pmx_conv_gather (first conv reading pillar rows through the cell map, no canvas)
vs pmx_conv on the scattered canvas: the same tcgen05 arithmetic on the same values,
so every output format must match BIT FOR BIT (int8 and f16, stride 1 and 2, ragged
tiles, empty frames, a full-size KITTI frame)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # (h, w), stride, batch, occupancy, pcap
    ((40, 36), 2, 2, 0.10, 400),
    ((38, 46), 2, 1, 0.30, 600),     # ragged tiles in both directions
    ((20, 18), 1, 2, 0.15, 200),
    ((21, 13), 1, 1, 0.50, 200),
    ((24, 16), 2, 1, 1.00, 400),     # every cell occupied (dense-tile path)
    ((496, 432), 2, 1, 0.075, 16000),  # KITTI blocks.0.0
    ((40, 36), 2, 2, 0.0, 16),        # empty frames
]


def _canvas_and_map(rng, batch, h, w, occ, pcap, cin, np_dt):
    cmap = np.zeros((batch, h, w), np.int32)  # slot + 1, 0 = empty
    feats = np.zeros((batch, pcap, cin), np_dt)
    canvas = np.zeros((batch, h, w, cin), np_dt)
    for b in range(batch):
        n = min(int(occ * h * w), pcap)
        cells = np.sort(rng.choice(h * w, size=n, replace=False))
        slots = np.arange(n, dtype=np.int32)
        if np_dt == np.int8:
            f = rng.integers(-128, 128, size=(n, cin), dtype=np.int8)
        else:
            f = rng.normal(size=(n, cin)).astype(np.float16)
        feats[b, :n] = f
        cmap[b].reshape(-1)[cells] = slots + 1
        canvas[b].reshape(-1, cin)[cells] = f
    return canvas, feats, cmap


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0][0]}x{c[0][1]}s{c[1]}b{c[2]}o{c[3]}")
@pytest.mark.parametrize("prec", ["int8", "fp16"])
def test_gather_matches_canvas(case, prec):
    import torch

    from paper_2601_12638_b200 import _native as N

    (h, w), s, batch, occ, pcap = case
    if s == 2 and (h % 2 or w % 2):
        h, w = h + h % 2, w + w % 2
    lib = N.load()
    rng = np.random.default_rng(h * 31 + w + s)
    cin, cout = 64, 64
    np_dt = np.int8 if prec == "int8" else np.float16
    canvas, feats, cmap = _canvas_and_map(rng, batch, h, w, occ, pcap, cin, np_dt)
    oh, ow = (h - 1) // s + 1, (w - 1) // s + 1
    desc = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.DTYPE_CODE[prec], batch=batch, in_h=h, in_w=w, in_c=cin,
                      in_c_stride=cin, in_c_offset=0, out_c=cout, k_h=3, k_w=3, stride_h=s, stride_w=s, pad_h=1,
                      pad_w=1, out_h=oh, out_w=ow, relu=1)
    if prec == "int8":
        wt = torch.from_numpy(rng.integers(-128, 128, size=(cout, 9 * cin), dtype=np.int8)).cuda()
        alpha = torch.from_numpy((rng.uniform(0.5, 2.0, cout) * 1e-4).astype(np.float32)).cuda()
    else:
        wt = torch.from_numpy((rng.normal(size=(cout, 9 * cin)) / 24.0).astype(np.float16)).cuda()
        alpha = None
    bias = torch.from_numpy(rng.normal(scale=0.1, size=cout).astype(np.float32)).cuda()
    x = torch.from_numpy(canvas).cuda()
    f = torch.from_numpy(feats).cuda()
    m = torch.from_numpy(cmap).cuda()
    spec = [(N.PMX_I8, 0.013), (N.PMX_F16, 0.0), (N.PMX_F32, 0.0)]

    def outs():
        bufs, lst = [], []
        for dt, sc in spec:
            t = torch.full((batch, oh, ow, cout), 7, dtype={N.PMX_F32: torch.float32, N.PMX_F16: torch.float16,
                                                            N.PMX_I8: torch.int8}[dt], device="cuda")
            bufs.append(t)
            lst.append(N.Out(ptr=t.data_ptr(), scale=sc, dtype=dt, c_stride=cout, c_offset=0))
        return bufs, N.outs_array(lst)

    keys_a = torch.empty(2, dtype=torch.int32, device="cuda")
    keys_b = torch.empty(2, dtype=torch.int32, device="cuda")
    N.check(lib.pmx_minmax_init(keys_a.data_ptr(), 1, N.stream_ptr()))
    N.check(lib.pmx_minmax_init(keys_b.data_ptr(), 1, N.stream_ptr()))
    ref, (arr, n) = outs()
    N.check(lib.pmx_conv(ctypes.byref(desc), x.data_ptr(), wt.data_ptr(), N.ptr(alpha), bias.data_ptr(), None, arr,
                         n, keys_a.data_ptr(), None, 0, N.stream_ptr()), "conv")
    got, (arr2, n2) = outs()
    N.check(lib.pmx_conv_gather(ctypes.byref(desc), f.data_ptr(), m.data_ptr(), pcap, wt.data_ptr(), N.ptr(alpha),
                                bias.data_ptr(), None, arr2, n2, keys_b.data_ptr(), N.stream_ptr()), "conv_gather")
    torch.cuda.synchronize()
    for a, b in zip(got, ref):
        assert torch.equal(a, b), (a.float() - b.float()).abs().max()
    assert torch.equal(keys_a, keys_b)


def test_gather_support_rules():
    """Shapes outside the gather kernels are reported (the engine then scatters a canvas)."""
    from paper_2601_12638_b200 import _native as N

    lib = N.load()

    def desc(h, w, s, cin, prec="int8", k=3):
        return N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.DTYPE_CODE[prec], batch=1, in_h=h, in_w=w, in_c=cin,
                          in_c_stride=cin, in_c_offset=0, out_c=64, k_h=k, k_w=k, stride_h=s, stride_w=s,
                          pad_h=k // 2, pad_w=k // 2, out_h=(h - 1) // s + 1, out_w=(w - 1) // s + 1, relu=1)

    assert lib.pmx_conv_gather_supported(ctypes.byref(desc(496, 432, 2, 64)))
    assert lib.pmx_conv_gather_supported(ctypes.byref(desc(496, 432, 2, 64, "fp16")))
    assert lib.pmx_conv_gather_supported(ctypes.byref(desc(20, 18, 1, 64)))
    assert not lib.pmx_conv_gather_supported(ctypes.byref(desc(496, 432, 2, 64, "fp32")))
    assert not lib.pmx_conv_gather_supported(ctypes.byref(desc(496, 432, 1, 64, k=1)))  # 1x1


def test_gather_single_int8_consumer_full_size():
    """The OUTK=1 fast epilogue (one int8 consumer) on the full KITTI stride-2 layer."""
    import torch

    from paper_2601_12638_b200 import _native as N

    lib = N.load()
    rng = np.random.default_rng(5)
    h, w, cin, cout, batch, pcap = 496, 432, 64, 64, 2, 16000
    canvas, feats, cmap = _canvas_and_map(rng, batch, h, w, 0.07, pcap, cin, np.int8)
    desc = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.PMX_I8, batch=batch, in_h=h, in_w=w, in_c=cin, in_c_stride=cin,
                      in_c_offset=0, out_c=cout, k_h=3, k_w=3, stride_h=2, stride_w=2, pad_h=1, pad_w=1,
                      out_h=248, out_w=216, relu=1)
    wt = torch.from_numpy(rng.integers(-128, 128, size=(cout, 9 * cin), dtype=np.int8)).cuda()
    alpha = torch.from_numpy((rng.uniform(0.5, 2.0, cout) * 1e-4).astype(np.float32)).cuda()
    bias = torch.from_numpy(rng.normal(scale=0.1, size=cout).astype(np.float32)).cuda()
    ys = []
    for gather in (False, True):
        y = torch.zeros((batch, 248, 216, cout), dtype=torch.int8, device="cuda")
        arr, n = N.outs_array([N.Out(ptr=y.data_ptr(), scale=0.02, dtype=N.PMX_I8, c_stride=cout, c_offset=0)])
        if gather:
            N.check(lib.pmx_conv_gather(ctypes.byref(desc), torch.from_numpy(feats).cuda().data_ptr(),
                                        torch.from_numpy(cmap).cuda().data_ptr(), pcap, wt.data_ptr(),
                                        alpha.data_ptr(), bias.data_ptr(), None, arr, n, None, N.stream_ptr()))
        else:
            xx = torch.from_numpy(canvas).cuda()
            N.check(lib.pmx_conv(ctypes.byref(desc), xx.data_ptr(), wt.data_ptr(), alpha.data_ptr(),
                                 bias.data_ptr(), None, arr, n, None, None, 0, N.stream_ptr()))
        torch.cuda.synchronize()
        ys.append(y)
    assert torch.equal(ys[0], ys[1])
    assert int((ys[0] != 0).sum()) > 0
