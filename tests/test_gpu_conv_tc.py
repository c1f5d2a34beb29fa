"""tcgen05 implicit-GEMM kernel vs the SIMT kernel on every PointPillars layer class.

INT8: the int32 accumulators are exact in both kernels and the epilogue formula is
identical, so every output format (int8 codes, f16, f32) must match BIT FOR BIT.
FP16: f16 x f16 products are exact; only the f32 summation order differs (<= 1e-5 rel).
Also checks the kernel is really the tcgen05 one (pmx_conv_backend)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # kind, cin, cout, k, stride, (h, w), batch
    ("conv", 64, 64, 3, 2, (40, 36), 2),     # blocks.0.0 (s2, Cin 64 int8 -> SW64)
    ("conv", 64, 64, 3, 1, (20, 18), 1),     # blocks.0.x
    ("conv", 64, 128, 3, 2, (20, 18), 1),    # blocks.1.0
    ("conv", 128, 128, 3, 1, (21, 13), 2),   # blocks.1.x (ragged tiles)
    ("conv", 128, 256, 3, 2, (12, 10), 1),   # blocks.2.0
    ("conv", 256, 256, 3, 1, (7, 9), 1),     # blocks.2.x
    ("deconv", 64, 128, 1, 1, (9, 7), 1),    # deblocks.0
    ("deconv", 128, 128, 2, 2, (6, 5), 2),   # deblocks.1
    ("deconv", 256, 128, 4, 4, (3, 4), 1),   # deblocks.2
    ("conv", 384, 4, 1, 1, (11, 13), 1),     # conv_dir_cls
    ("conv", 384, 14, 1, 1, (11, 13), 1),    # conv_reg
    ("conv", 384, 2, 1, 1, (11, 13), 1),     # conv_cls
    ("conv", 384, 20, 1, 1, (248, 216), 1),  # fused heads, full size
    ("conv", 64, 64, 3, 2, (496, 432), 1),   # blocks.0.0 full size
    ("conv", 128, 128, 3, 1, (124, 108), 1), # blocks.1.x full size, batch 1
    ("conv", 256, 256, 3, 1, (62, 54), 1),   # blocks.2.x full size, batch 1 (N split to 4 x 64)
    ("deconv", 256, 128, 4, 4, (62, 54), 1), # deblocks.2 full size, batch 1
] + [  # 2-CTA clusters (cta_group::2, M = 256): enough tiles for the pair plan
    ("conv", 256, 256, 3, 1, (62, 54), 12),  # blocks.2.x full size, batch 12 (324 tiles)
    ("conv", 128, 256, 3, 2, (124, 108), 12),# blocks.2.0 full size, batch 12
    ("conv", 256, 256, 3, 1, (61, 37), 17),  # 323 pixel tiles: the last pair's rank 1 idles
    ("conv", 128, 128, 3, 1, (124, 108), 4), # blocks.1.x: pair plan in the nohalo mode
]
CLUSTER_CASES = CASES[-4:]


def _run(lib, N, torch, desc, x, w, alpha, bias, outs_spec, mode, observe=True):
    outs = []
    bufs = []
    for dt, scale in outs_spec:
        t = torch.zeros((desc.batch, desc.out_h, desc.out_w, desc.out_c),
                        dtype={N.PMX_F32: torch.float32, N.PMX_F16: torch.float16, N.PMX_I8: torch.int8}[dt],
                        device="cuda")
        bufs.append(t)
        outs.append(N.Out(ptr=t.data_ptr(), scale=scale, dtype=dt, c_stride=desc.out_c, c_offset=0))
    arr, n = N.outs_array(outs)
    lib.pmx_set_conv_backend(mode)
    keys = torch.empty(2, dtype=torch.int32, device="cuda")
    N.check(lib.pmx_minmax_init(keys.data_ptr(), 1, N.stream_ptr()))
    try:
        N.check(lib.pmx_conv(ctypes.byref(desc), x.data_ptr(), w.data_ptr(), None if alpha is None else alpha.data_ptr(),
                             bias.data_ptr(), None, arr, n, keys.data_ptr() if observe else None, None, 0,
                             N.stream_ptr()), "conv")
        torch.cuda.synchronize()
    finally:
        lib.pmx_set_conv_backend(0)
    return bufs, N.decode_keys(keys.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}x{c[2]}k{c[3]}s{c[4]}_{c[5][0]}x{c[5][1]}")
@pytest.mark.parametrize("prec", ["int8", "fp16"])
@pytest.mark.parametrize("tc_mode", [0, 2], ids=["auto", "nohalo"])
def test_tcgen05_matches_simt(case, prec, tc_mode):
    import torch

    from paper_2601_12638_b200 import _native as N

    lib = N.load()
    kind, cin, cout, k, s, (h, w), batch = case
    rng = np.random.default_rng(cin * 7 + cout + k + s + h)
    deconv = kind == "deconv"
    if deconv:
        oh, ow = h * s, w * s
        ngemm = k * k * cout
        wshape = (ngemm, cin)
    else:
        pad = 1 if k == 3 else 0
        oh, ow = (h + 2 * pad - k) // s + 1, (w + 2 * pad - k) // s + 1
        wshape = (cout, k * k * cin)
    desc = N.ConvDesc(kind=N.PMX_DECONV2D if deconv else N.PMX_CONV2D, in_dtype=N.DTYPE_CODE[prec], batch=batch,
                      in_h=h, in_w=w, in_c=cin, in_c_stride=cin, in_c_offset=0, out_c=cout, k_h=k, k_w=k,
                      stride_h=s, stride_w=s, pad_h=0 if deconv or k == 1 else 1, pad_w=0 if deconv or k == 1 else 1,
                      out_h=oh, out_w=ow, relu=1)
    if prec == "int8":
        x = torch.from_numpy(rng.integers(-128, 128, size=(batch, h, w, cin), dtype=np.int8)).cuda()
        wt = torch.from_numpy(rng.integers(-128, 128, size=wshape, dtype=np.int8)).cuda()
        alpha = torch.from_numpy((rng.uniform(0.5, 2.0, cout) * 1e-4).astype(np.float32)).cuda()
    else:
        x = torch.from_numpy(rng.normal(size=(batch, h, w, cin)).astype(np.float16)).cuda()
        wt = torch.from_numpy((rng.normal(size=wshape) / np.sqrt(wshape[1])).astype(np.float16)).cuda()
        alpha = None
    bias = torch.from_numpy(rng.normal(scale=0.1, size=cout).astype(np.float32)).cuda()
    spec = [(N.PMX_F32, 0.0), (N.PMX_I8, 0.013), (N.PMX_F16, 0.0)]
    assert lib.pmx_conv_backend(desc.in_dtype, desc.kind).decode() == "tcgen05"
    tc, ktc = _run(lib, N, torch, desc, x, wt, alpha, bias, spec, tc_mode)
    ref, kref = _run(lib, N, torch, desc, x, wt, alpha, bias, spec, 1)
    if prec == "int8":
        for a, b in zip(tc, ref):
            assert torch.equal(a, b), (a.float() - b.float()).abs().max()
        np.testing.assert_array_equal(ktc, kref)
    else:
        a, b = tc[0].double(), ref[0].double()
        assert float((a - b).norm() / b.norm()) <= 1e-5
        codes = (tc[1].int() - ref[1].int()).abs()
        assert int(codes.max()) <= 1 and float((codes != 0).float().mean()) < 1e-3


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}x{c[2]}k{c[3]}s{c[4]}_{c[5][0]}x{c[5][1]}")
@pytest.mark.parametrize("relu", [1, 0])
def test_tcgen05_single_int8_consumer(case, relu):
    """The OUTK=1 epilogue (one 16-byte aligned int8 consumer: the clamp-free fast
    quantizer with the byte-permute ReLU, and its exact fallback) vs the SIMT kernel,
    bit for bit, with scales chosen so that codes saturate and hit exact .5 ties."""
    import torch

    from paper_2601_12638_b200 import _native as N

    lib = N.load()
    kind, cin, cout, k, s, (h, w), batch = case
    if cout % 16:
        pytest.skip("OUTK=1 needs 16-byte aligned rows")
    rng = np.random.default_rng(cin * 11 + cout + k + s + h + relu)
    deconv = kind == "deconv"
    if deconv:
        oh, ow, wshape = h * s, w * s, (k * k * cout, cin)
    else:
        pad = 1 if k == 3 else 0
        oh, ow, wshape = (h + 2 * pad - k) // s + 1, (w + 2 * pad - k) // s + 1, (cout, k * k * cin)
    desc = N.ConvDesc(kind=N.PMX_DECONV2D if deconv else N.PMX_CONV2D, in_dtype=N.PMX_I8, batch=batch, in_h=h,
                      in_w=w, in_c=cin, in_c_stride=cin, in_c_offset=0, out_c=cout, k_h=k, k_w=k, stride_h=s,
                      stride_w=s, pad_h=0 if deconv or k == 1 else 1, pad_w=0 if deconv or k == 1 else 1,
                      out_h=oh, out_w=ow, relu=relu)
    x = torch.from_numpy(rng.integers(-128, 128, size=(batch, h, w, cin), dtype=np.int8)).cuda()
    wt = torch.from_numpy(rng.integers(-128, 128, size=wshape, dtype=np.int8)).cuda()
    # alpha = 2^-12: y = acc / 4096 + bias, with bias multiples of 1/8 and scale 1/2
    # many y/s land exactly on .5 ties; the wide accumulator range saturates codes
    kdim = wshape[1]
    alpha = torch.full((cout,), 2.0 ** (-9 if kdim <= 128 else -12), dtype=torch.float32, device="cuda")
    bias = torch.from_numpy((rng.integers(-8, 8, cout) / 8.0).astype(np.float32)).cuda()
    outs = []
    for mode in (0, 1):
        y = torch.full((batch, oh, ow, cout), 99, dtype=torch.int8, device="cuda")
        arr, n = N.outs_array([N.Out(ptr=y.data_ptr(), scale=0.5, dtype=N.PMX_I8, c_stride=cout, c_offset=0)])
        lib.pmx_set_conv_backend(mode)
        try:
            N.check(lib.pmx_conv(ctypes.byref(desc), x.data_ptr(), wt.data_ptr(), alpha.data_ptr(), bias.data_ptr(),
                                 None, arr, n, None, None, 0, N.stream_ptr()), "conv")
            torch.cuda.synchronize()
        finally:
            lib.pmx_set_conv_backend(0)
        outs.append(y)
    assert torch.equal(outs[0], outs[1]), (outs[0].int() - outs[1].int()).abs().max()
    c = outs[0].int()
    assert int((c == 127).sum()) > 0 and int((c != 0).sum()) > 0
    if relu:
        assert int(c.min()) == 0
    else:
        assert int(c.min()) < 0


PAIR_CASES = [  # the (int8, f16) consumer pair of a block's last conv: staged f16 stores
    ("conv", 64, 64, 3, 1, (20, 18), 2),      # blocks.0.9 shape class (4 KB/warp staging)
    ("conv", 64, 64, 3, 1, (248, 216), 1),    # blocks.0.9 full size
    ("conv", 128, 128, 3, 1, (21, 13), 2),    # blocks.1.15 (1 KB/warp staging next to the halo)
    ("conv", 128, 128, 3, 1, (124, 108), 1),  # blocks.1.15 full size
    ("conv", 256, 256, 3, 1, (7, 9), 1),      # blocks.2.x class
]


@pytest.mark.parametrize("case", PAIR_CASES, ids=lambda c: f"{c[0]}{c[1]}x{c[2]}k{c[3]}s{c[4]}_{c[5][0]}x{c[5][1]}")
@pytest.mark.parametrize("order", ["i8f16", "f16i8"])
def test_tcgen05_int8_f16_pair(case, order):
    """Two consumers (int8 codes + binary16), no observer: the staged-store epilogue
    (and its small-staging mode) vs the SIMT kernel, bit for bit (int8 arithmetic)."""
    import torch

    from paper_2601_12638_b200 import _native as N

    lib = N.load()
    kind, cin, cout, k, s, (h, w), batch = case
    rng = np.random.default_rng(cin * 5 + cout + h)
    oh, ow = (h + 2 - k) // s + 1, (w + 2 - k) // s + 1
    desc = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.PMX_I8, batch=batch, in_h=h, in_w=w, in_c=cin, in_c_stride=cin,
                      in_c_offset=0, out_c=cout, k_h=k, k_w=k, stride_h=s, stride_w=s, pad_h=1, pad_w=1, out_h=oh,
                      out_w=ow, relu=1)
    x = torch.from_numpy(rng.integers(-128, 128, size=(batch, h, w, cin), dtype=np.int8)).cuda()
    wt = torch.from_numpy(rng.integers(-128, 128, size=(cout, k * k * cin), dtype=np.int8)).cuda()
    alpha = torch.from_numpy((rng.uniform(0.5, 2.0, cout) * 1e-4).astype(np.float32)).cuda()
    bias = torch.from_numpy(rng.normal(scale=0.1, size=cout).astype(np.float32)).cuda()
    spec = [(N.PMX_I8, 0.013), (N.PMX_F16, 0.0)]
    if order == "f16i8":
        spec = spec[::-1]
    tc, _ = _run(lib, N, torch, desc, x, wt, alpha, bias, spec, 0, observe=False)
    ref, _ = _run(lib, N, torch, desc, x, wt, alpha, bias, spec, 1, observe=False)
    for a, b in zip(tc, ref):
        assert torch.equal(a, b), (a.float() - b.float()).abs().max()


@pytest.mark.parametrize("case", CLUSTER_CASES, ids=lambda c: f"{c[1]}x{c[2]}s{c[4]}_{c[5][0]}x{c[5][1]}b{c[6]}")
def test_pair_plan_selected(case):
    """The CLUSTER_CASES really run the 2-CTA plan (bit 1 of pmx_conv_tc_supported), so the
    parity tests above cover it; PMX_PAIR=0 is the only way to turn it off."""
    from paper_2601_12638_b200 import _native as N

    lib = N.load()
    kind, cin, cout, k, s, (h, w), batch = case
    oh, ow = (h + 2 - 3) // s + 1, (w + 2 - 3) // s + 1
    desc = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.PMX_I8, batch=batch, in_h=h, in_w=w, in_c=cin, in_c_stride=cin,
                      in_c_offset=0, out_c=cout, k_h=3, k_w=3, stride_h=s, stride_w=s, pad_h=1, pad_w=1, out_h=oh,
                      out_w=ow, relu=1)
    lib.pmx_set_conv_backend(2 if cout == 128 else 0)
    try:
        code = lib.pmx_conv_tc_supported(ctypes.byref(desc))
    finally:
        lib.pmx_set_conv_backend(0)
    assert code & 1 and code & 2, code
    assert (code >> 2) & 3 == 0  # the per-tap TMA ring (pairs are never planned for halo / GEMM)


def test_halo_pair_opt_in_bit_exact():
    """The opt-in 2-CTA halo path (PMX_HALO_PAIR=1, read once per process: a subprocess)
    is planned for large int8 halo layers and matches the SIMT kernel bit for bit."""
    import os
    import subprocess
    import sys

    code = r'''
import ctypes, numpy as np, torch
from paper_2601_12638_b200 import _native as N
lib = N.load()
for (cin, cout, s, h, w, b) in [(64, 64, 1, 248, 216, 2), (64, 64, 2, 496, 432, 1), (128, 128, 1, 124, 108, 4)]:
    oh, ow = (h - 1) // s + 1, (w - 1) // s + 1
    d = N.ConvDesc(kind=N.PMX_CONV2D, in_dtype=N.PMX_I8, batch=b, in_h=h, in_w=w, in_c=cin, in_c_stride=cin,
                   in_c_offset=0, out_c=cout, k_h=3, k_w=3, stride_h=s, stride_w=s, pad_h=1, pad_w=1, out_h=oh,
                   out_w=ow, relu=1)
    plan = lib.pmx_conv_tc_supported(ctypes.byref(d))
    assert plan & 2 and (plan >> 2) & 3 == 2, plan
    rng = np.random.default_rng(cin + s + h)
    x = torch.from_numpy(rng.integers(-128, 128, size=(b, h, w, cin), dtype=np.int8)).cuda()
    wt = torch.from_numpy(rng.integers(-128, 128, size=(cout, 9 * cin), dtype=np.int8)).cuda()
    alpha = torch.full((cout,), 2.0 ** -12, device="cuda")
    bias = torch.from_numpy((rng.integers(-8, 8, cout) / 8.0).astype(np.float32)).cuda()
    outs = []
    for mode in (0, 1):
        y = torch.zeros((b, oh, ow, cout), dtype=torch.int8, device="cuda")
        arr, n = N.outs_array([N.Out(ptr=y.data_ptr(), scale=0.5, dtype=N.PMX_I8, c_stride=cout, c_offset=0)])
        lib.pmx_set_conv_backend(mode)
        N.check(lib.pmx_conv(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), alpha.data_ptr(), bias.data_ptr(), None,
                             arr, n, None, None, 0, N.stream_ptr()))
        torch.cuda.synchronize()
        lib.pmx_set_conv_backend(0)
        outs.append(y)
    assert torch.equal(outs[0], outs[1]), (cin, s)
print("halo pair ok")
'''
    env = dict(os.environ, PMX_HALO_PAIR="1", PMX_NO_BUILD="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parent.parent))
    assert r.returncode == 0 and "halo pair ok" in r.stdout, r.stdout + r.stderr
