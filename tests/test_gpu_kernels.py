"""T0 parity of the element-wise / index kernels against the oracle and the reference's
golden vectors: quantize codes, fake_quant, fp16, observers, pillarize, top-k."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import pillars_oracle as O
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


def test_quantize_golden_bit_exact(pm, golden):
    g = golden("ref_quant.npz")
    i = 0
    while f"x{i}" in g:
        qp = pm.QuantParams(scale=float(g[f"scale{i}"]))
        np.testing.assert_array_equal(pm.quantize(g[f"x{i}"], qp), g[f"codes{i}"])
        np.testing.assert_array_equal(pm.fake_quant(g[f"x{i}"], qp), g[f"fq{i}"])
        i += 1


def test_quantize_near_ties_bit_exact(pm):
    """f32 estimates alone mismatch ~30% of near-tie codes; the guard band must fix all."""
    rng = np.random.default_rng(7)
    for s in (0.0123456789, 0.37, 1.0 / 3.0, 2.54 / 127.0, 5.5):
        k = rng.integers(-140, 140, size=1_000_000)
        x = ((k + 0.5) * s * (1.0 + rng.normal(scale=3e-7, size=k.size))).astype(np.float32)
        x = np.concatenate([x, np.nextafter(x, np.inf), np.nextafter(x, -np.inf)])
        np.testing.assert_array_equal(pm.quantize(x, pm.QuantParams(scale=s)), O.quantize(x, s))
        y = rng.normal(scale=50 * s, size=2_000_000).astype(np.float32)
        np.testing.assert_array_equal(pm.quantize(y, pm.QuantParams(scale=s)), O.quantize(y, s))


def test_reference_quant_known_answers(pm):
    qp = pm.QuantParams(scale=1.0)
    assert [pm.quantize(v, qp) for v in (2.5, 3.5, -2.5, 1000.0, -1000.0)] == [2, 4, -2, 127, -128]
    qp = pm.QuantParams(scale=0.03125)
    t = np.arange(-127, 128, dtype=np.float32) * np.float32(0.03125)
    np.testing.assert_array_equal(pm.fake_quant(t, qp), t)
    assert pm.fp16_roundtrip(np.float32(2049.0)) == 2048.0
    assert pm.fp16_roundtrip(np.float32(1e6)) == 65504.0
    np.testing.assert_array_equal(pm.fp16_roundtrip(np.array([1e30, -1e30, 65519.0], np.float32)),
                                  [65504.0, -65504.0, 65504.0])
    ints = np.arange(-2048, 2049, dtype=np.float32)
    np.testing.assert_array_equal(pm.fp16_roundtrip(ints), ints)
    obs = pm.observe(pm.MinMaxObserver(), np.array([-0.5, 2.54]))
    assert obs.quant_params().scale == 2.54 / 127.0
    with pytest.raises(ValueError, match="non-finite"):
        pm.observe(pm.MinMaxObserver(), np.array([1.0, np.nan], np.float32))


def test_fp16_golden_and_weight_quant(pm, golden):
    g = golden("ref_quant.npz")
    np.testing.assert_array_equal(pm.fp16_roundtrip(g["fp16_in"]), g["fp16_out"])
    qp = pm.weight_quant_params(g["w"], per_channel=True)
    np.testing.assert_array_equal(pm.fake_quant_per_channel(g["w"], qp), g["w_fq_pc"])
    codes = pm.quant.weight_codes(g["w"], qp).cpu().numpy()
    np.testing.assert_array_equal(codes, O.weight_codes_per_channel(g["w"], qp.scales))


def _rne_f16_bits(u):
    """Independent integer model of clip(+-65504) + round-to-nearest-even f32 -> f16.

    u: int64 tensor of f32 bit patterns.  Returns (f16 bits, is_nan)."""
    import torch

    sign = (u >> 31) & 1
    e = (u >> 23) & 0xFF
    m = u & 0x7FFFFF
    mant = m | 0x800000
    ue = e - 127
    one = torch.ones_like(u)

    def rne_shift(v, sh):
        q = v >> sh
        rem = v - (q << sh)
        half = one << (sh - 1)
        up = (rem > half) | ((rem == half) & ((q & 1) == 1))
        return q + up.to(v.dtype)

    normal = ((ue + 15) << 10) + rne_shift(mant, torch.full_like(u, 13)) - 1024
    sub = rne_shift(mant, (-ue - 1).clamp(14, 40))
    bits = torch.where(ue >= -14, normal, sub)
    bits = torch.where(e == 0, torch.zeros_like(bits), bits)
    big = (ue > 15) | ((ue == 15) & (m > (0x3FF << 13)))
    bits = torch.where(big | (e == 0xFF), torch.full_like(bits, 0x7BFF), bits)
    nan = (e == 0xFF) & (m != 0)
    return (sign << 15) | bits, nan


def test_fp16_exhaustive_all_f32_bit_patterns(pm):
    """All 2^32 f32 inputs: the device cast vs an independent integer RNE model."""
    import torch

    from paper_2601_12638_b200 import _native as N

    lib = N.load()
    chunk = 1 << 28
    for c in range(1 << 4):
        u = torch.arange(c * chunk, (c + 1) * chunk, dtype=torch.int64, device="cuda")
        x = (u - (u >= (1 << 31)).long() * (1 << 32)).to(torch.int32).view(torch.float32)
        out = torch.empty(chunk, dtype=torch.float16, device="cuda")
        N.check(lib.pmx_fp16_roundtrip(x.data_ptr(), chunk, None, out.data_ptr(), N.stream_ptr()))
        got = out.view(torch.int16).to(torch.int64) & 0xFFFF
        want, nan = _rne_f16_bits(u)
        ok = (got == want) | (nan & ((got & 0x7C00) == 0x7C00) & ((got & 0x3FF) != 0))
        bad = (~ok).nonzero()
        assert bad.numel() == 0, (c, hex(int(u[bad[0]])), hex(int(got[bad[0]])), hex(int(want[bad[0]])))
        del u, x, out, got, want, nan, ok


def test_minmax_observer_exact(pm):
    rng = np.random.default_rng(3)
    for n in (1, 31, 1000, 1_000_003):
        x = rng.normal(size=n).astype(np.float32)
        assert pm.quant.device_minmax(x) == (float(x.min()), float(x.max()))


# ----------------------------------------------------------------------------- pillarize


def test_pillarize_toy_golden_bit_exact(pm, golden):
    g = golden("ref_toy.npz")
    meta = json.loads((GOLDEN / "ref_toy_meta.json").read_text())
    det = meta["detector"]
    for i in range(meta["n_samples"]):
        s = pm.pillarize(pm.Scene(points=g[f"pts{i}"]), tuple(det["grid"]), det["max_points_per_pillar"],
                         det["field_size"])
        np.testing.assert_array_equal(s.coords, g[f"coords{i}"])
        np.testing.assert_array_equal(s.point_mask, g[f"mask{i}"])
        np.testing.assert_array_equal(s.features, g[f"feat{i}"])


def _kitti_case(pm, n, seed, cfg, clustered=False):
    pts = pm.make_frame(n, seed, cfg)
    if clustered:  # many points per cell: exercises the M=32 truncation and > 32-point cells
        rng = np.random.default_rng(seed)
        c = pts[: n // 4].copy()
        c[:, 0] = cfg.x_range[0] + 1.0 + rng.uniform(0, 0.3, len(c))
        c[:, 1] = cfg.y_range[0] + 1.0 + rng.uniform(0, 0.5, len(c))
        pts = np.concatenate([pts, c]).astype(np.float32)
        pts = pts[rng.permutation(len(pts))]
    return pts


@pytest.mark.parametrize("n,max_pillars,clustered", [
    (3000, 1500, False), (3000, 50000, False), (4000, 800, True), (1, 10, False), (0, 10, False),
])
def test_pillarize_kitti_vs_oracle(pm, n, max_pillars, clustered):
    cfg = pm.PointPillarsConfig.small(max_pillars=max_pillars)
    pts = _kitti_case(pm, n, 11, cfg, clustered) if n else np.zeros((0, 4), np.float32)
    spec = cfg.grid_spec()
    got = pm.scenes.pillar_index(pts, spec)
    flat = O.bin_points(pts[:, :2], spec.grid, spec.origin, spec.cell)
    want = O.pillar_index(flat, spec.grid, spec.max_points, spec.max_pillars)
    P = len(want.coords)
    assert got["n_pillars"] == P
    np.testing.assert_array_equal(got["coords"], want.coords)
    np.testing.assert_array_equal(got["counts"], want.counts)
    np.testing.assert_array_equal(got["pt_idx"], want.pt_idx)
    if P:
        s = pm.pillarize_points(pts, spec)
        f, m = O.pillar_features9(pts, want, spec.origin, spec.cell)
        np.testing.assert_array_equal(s.features, f)
        np.testing.assert_array_equal(s.point_mask, m)


def test_pillarize_out_of_range_points_clamp(pm):
    cfg = pm.PointPillarsConfig.small(max_pillars=5000)
    pts = np.array([[-5.0, -30.0, 0, 0], [1e6, 1e6, 0, 0], [-0.01, 0.0, 0, 0], [7.679, 5.1199, 0, 0]], np.float32)
    spec = cfg.grid_spec()
    got = pm.scenes.pillar_index(pts, spec)
    want = O.pillar_index(O.bin_points(pts[:, :2], spec.grid, spec.origin, spec.cell), spec.grid, 32, 5000)
    np.testing.assert_array_equal(got["coords"], want.coords)
    np.testing.assert_array_equal(got["pt_idx"], want.pt_idx)


@pytest.mark.parametrize("sizes", [(3000, 0, 1, -4000, 2500),  # batch <= 8 (the persistent opt-in applies)
                                   (3000, 0, 1, -4000, 2500, 7, 3100, 2900, 0, 2000)])  # batch 10
def test_pillarize_batch_vs_oracle(pm, sizes):
    """Frames of one batched pmx_pillarize call (ragged, empty, clustered (negative
    size), capped) vs the oracle frame by frame."""
    import ctypes

    import torch

    from paper_2601_12638_b200 import _native as N

    lib = N.require_cuda()
    cfg = pm.PointPillarsConfig.small(max_pillars=900)
    spec = cfg.grid_spec()
    frames = [(_kitti_case(pm, abs(n), 40 + i, cfg, n < 0) if n else np.zeros((0, 4), np.float32))
              for i, n in enumerate(sizes)]
    B = len(frames)
    nmax = max(1, max(len(f) for f in frames))
    h, w = spec.grid
    pcap = spec.max_pillars
    g = spec.to_c()
    allp = np.concatenate(frames + [np.zeros((1, 4), np.float32)]).astype(np.float32)
    offs = np.concatenate([[0], np.cumsum([len(f) for f in frames])]).astype(np.int64)
    pts = torch.from_numpy(allp).cuda()
    offs_d = torch.from_numpy(offs).cuda()
    coords = torch.empty((B, pcap, 2), dtype=torch.int32, device="cuda")
    counts = torch.empty((B, pcap), dtype=torch.int32, device="cuda")
    pt_idx = torch.empty((B, pcap, spec.max_points), dtype=torch.int32, device="cuda")
    n_pil = torch.zeros((B,), dtype=torch.int32, device="cuda")
    ws_bytes = lib.pmx_pillarize_workspace(ctypes.byref(g), B, nmax)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):  # twice: the workspace is re-initialised by every call
        N.check(lib.pmx_pillarize(pts.data_ptr(), offs_d.data_ptr(), B, nmax, ctypes.byref(g), pcap,
                                  coords.data_ptr(), counts.data_ptr(), pt_idx.data_ptr(), n_pil.data_ptr(),
                                  ws.data_ptr(), ws_bytes, N.stream_ptr()), "pillarize")
    torch.cuda.synchronize()
    for b, f in enumerate(frames):
        want = O.pillar_index(O.bin_points(f[:, :2], spec.grid, spec.origin, spec.cell), spec.grid,
                              spec.max_points, pcap)
        P = len(want.coords)
        assert int(n_pil[b]) == P, (b, int(n_pil[b]), P)
        np.testing.assert_array_equal(coords[b, :P].cpu().numpy(), want.coords)
        np.testing.assert_array_equal(counts[b, :P].cpu().numpy(), want.counts)
        np.testing.assert_array_equal(pt_idx[b, :P].cpu().numpy(), want.pt_idx)


def test_pillarize_persistent_opt_in_subprocess(pm):
    """The opt-in one-kernel pillarize (PMX_PILLARIZE_PERSIST=1, cooperative launch with
    grid-wide barriers; read once per process: a subprocess) passes the batched parity."""
    import os
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, PMX_PILLARIZE_PERSIST="1", PMX_NO_BUILD="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        str(Path(__file__)) + "::test_pillarize_batch_vs_oracle"], env=env, cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "2 passed" in r.stdout, r.stdout[-2000:]


@pytest.mark.slow
@pytest.mark.parametrize("n,cap", [(20000, 12000), (120000, 16000), (150000, 16000)])
def test_pillarize_full_size(pm, n, cap):
    cfg = pm.PointPillarsConfig(max_pillars=cap)
    pts = pm.make_frame(n, 5, cfg, outlier_frac=0.01)
    spec = cfg.grid_spec()
    got = pm.scenes.pillar_index(pts, spec)
    want = O.pillar_index(O.bin_points(pts[:, :2], spec.grid, spec.origin, spec.cell), spec.grid, 32, cap)
    np.testing.assert_array_equal(got["coords"], want.coords)
    np.testing.assert_array_equal(got["counts"], want.counts)
    np.testing.assert_array_equal(got["pt_idx"], want.pt_idx)


# ----------------------------------------------------------------------------- decode


class _Geom:
    def __init__(self, spec):
        self.out_stride = spec.out_stride
        self.origin = spec.origin
        self.anchor_size = spec.anchor_size
        self.anchor_z = spec.anchor_z
        self.anchor_rotations = spec.rotations
        self.dir_offset = spec.dir_offset


@pytest.mark.parametrize("H,W,k,ties", [(248, 216, 100, False), (32, 24, 100, True), (8, 6, 200, False),
                                        (248, 216, 512, "const"), (248, 216, 100, "coarse"), (1, 1, 5, False)])
def test_decode_topk_exact_index_set(pm, H, W, k, ties):
    """Exact top-k: the shared-memory sort (few survivors of the histogram threshold)
    and the radix-select path (all 107k logits equal, or > 4096 in the k-th bin)."""
    spec = pm.PointPillarsConfig(topk=k).anchor_spec()
    rng = np.random.default_rng(H * W)
    A = len(spec.rotations)
    cls = rng.normal(size=(A, H, W)).astype(np.float32)
    if ties is True:
        cls = np.round(cls * 2) / 2  # many equal logits: ties resolve to the lower index
    elif ties == "const":
        cls[:] = 0.25
    elif ties == "coarse":
        cls = (3.0 + np.round(cls) / 64).astype(np.float32)  # thousands of keys share the k-th bin
    box = (0.1 * rng.normal(size=(7 * A, H, W))).astype(np.float32)
    dr = rng.normal(size=(2 * A, H, W)).astype(np.float32)
    out = pm.decode_topk(cls, box, dr, spec)
    kk = min(k, A * H * W)
    idx, logit, _, boxes, labels = O.decode_topk(cls, box, dr, _Geom(spec), kk)
    got_idx = out["idx"][0].cpu().numpy()[:kk]
    np.testing.assert_array_equal(got_idx, idx)
    np.testing.assert_array_equal(out["logit"][0].cpu().numpy()[:kk], logit)
    np.testing.assert_array_equal(out["dir"][0].cpu().numpy()[:kk], labels)
    np.testing.assert_allclose(out["boxes"][0].cpu().numpy()[:kk], boxes, rtol=2e-6, atol=2e-6)
    if kk < k:
        assert (out["idx"][0].cpu().numpy()[kk:] == -1).all()


# ----------------------------------------------------------------------------- PFN (K4)


@pytest.mark.parametrize("prec", ["int8", "fp16", "fp32"])
@pytest.mark.parametrize("clustered", [False, True])
def test_pfn_pillar_rows_vs_oracle(pm, prec, clustered):
    """pmx_pfn_pillars (the 9-feature PFN: transform -> linear -> bias -> ReLU -> max over
    points, one f32 row per pillar) vs a numpy restatement on the oracle's pillar
    features; clustered frames put up to 32 points in a pillar (the kernel keeps 8 per
    pillar in shared memory and rebuilds the rest)."""
    import ctypes

    import torch

    from paper_2601_12638_b200 import _native as N

    cfg = pm.PointPillarsConfig.small(max_pillars=800)
    pts = _kitti_case(pm, 4000, 21, cfg, clustered)
    spec = cfg.grid_spec()
    want_idx = O.pillar_index(O.bin_points(pts[:, :2], spec.grid, spec.origin, spec.cell), spec.grid, 32, 800)
    feats, mask = O.pillar_features9(pts, want_idx, spec.origin, spec.cell)
    P = len(want_idx.coords)
    assert (want_idx.counts.max() > 8) == clustered
    rng = np.random.default_rng(3)
    C = 64
    w = rng.normal(scale=0.3, size=(C, 9)).astype(np.float32)
    bias = rng.normal(scale=0.1, size=C).astype(np.float32)
    in_scale = float(np.abs(feats).max() / 127.0)
    if prec == "int8":
        xq = O.quantize(feats, in_scale).astype(np.float64)
        ws = np.abs(w).max(axis=1) / 127.0
        wq = np.rint(w.astype(np.float64) / ws[:, None]).clip(-128, 127)
        acc = np.einsum("pmj,cj->pmc", xq, wq)  # exact integers
        alpha = (in_scale * ws).astype(np.float32)
        y = (acc * alpha.astype(np.float64) + bias).astype(np.float32)
        wdev = torch.from_numpy(wq.astype(np.int8)).cuda()
        adev = torch.from_numpy(alpha).cuda()
    else:
        x = feats if prec == "fp32" else O.fp16_roundtrip(feats)
        wv = w if prec == "fp32" else O.fp16_roundtrip(w)
        y = (np.einsum("pmj,cj->pmc", x.astype(np.float64), wv.astype(np.float64)) + bias).astype(np.float32)
        wdev = torch.from_numpy(wv if prec == "fp32" else wv.astype(np.float16)).cuda()
        adev = None
    y = np.maximum(y, 0)
    y = np.where(mask[:, :, None], y, -np.inf).max(axis=1)  # [P, C]
    # device pipeline: pillarize -> PFN rows
    lib = N.load()
    g = spec_c = pm.engine.GridSpec(grid=spec.grid, origin=spec.origin, cell=spec.cell, max_points=32,
                                    max_pillars=800).to_c()
    dpts = torch.from_numpy(pts).cuda()
    offs = torch.tensor([0, len(pts)], dtype=torch.int64, device="cuda")
    coords = torch.empty((1, 800, 2), dtype=torch.int32, device="cuda")
    counts = torch.empty((1, 800), dtype=torch.int32, device="cuda")
    pt_idx = torch.empty((1, 800, 32), dtype=torch.int32, device="cuda")
    npil = torch.empty((1,), dtype=torch.int32, device="cuda")
    wsb = lib.pmx_pillarize_workspace(ctypes.byref(g), 1, len(pts))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(lib.pmx_pillarize(dpts.data_ptr(), offs.data_ptr(), 1, len(pts), ctypes.byref(g), 800, coords.data_ptr(),
                              counts.data_ptr(), pt_idx.data_ptr(), npil.data_ptr(), ws.data_ptr(), wsb,
                              N.stream_ptr()), "pillarize")
    rows = torch.full((800, C), -7.0, dtype=torch.float32, device="cuda")
    arr, n = N.outs_array([N.Out(ptr=rows.data_ptr(), scale=0.0, dtype=N.PMX_F32, c_stride=C, c_offset=0)])
    d = N.PfnDesc(source=N.PMX_PFN_FROM_POINTS9, in_dtype=N.DTYPE_CODE[prec], n_features=9, channels=C,
                  max_points=32, relu=1, in_scale=in_scale if prec == "int8" else 0.0)
    bdev = torch.from_numpy(bias).cuda()
    N.check(lib.pmx_pfn_pillars(ctypes.byref(d), ctypes.byref(g), 1, 800, dpts.data_ptr(), offs.data_ptr(), None,
                                None, coords.data_ptr(), counts.data_ptr(), pt_idx.data_ptr(), npil.data_ptr(),
                                wdev.data_ptr(), N.ptr(adev), bdev.data_ptr(), None, arr, n, None, None,
                                N.stream_ptr()), "pfn_pillars")
    got = rows.cpu().numpy()
    assert int(npil.item()) == P
    np.testing.assert_allclose(got[:P], y, rtol=1e-5, atol=1e-5)
    assert (got[P:] == -7.0).all()  # rows past n_pillars untouched


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_pfn_every_live_pillar_count(pm, prec):
    """Regression: the PFN's pillar-pair loop used a full-warp shuffle after a divergent
    branch, so a warp whose last live pillar sat in the first half of a pair wrote its row
    at a garbage address.  Every n_pillars from 1 to 70 (and the full count), dense clusters
    included, must give the reference rows and leave the rest untouched."""
    import ctypes

    import torch

    from paper_2601_12638_b200 import _native as N

    cfg = pm.PointPillarsConfig.small(max_pillars=800)
    pts = _kitti_case(pm, 4000, 23, cfg, True)
    spec = cfg.grid_spec()
    idx = O.pillar_index(O.bin_points(pts[:, :2], spec.grid, spec.origin, spec.cell), spec.grid, 32, 800)
    feats, mask = O.pillar_features9(pts, idx, spec.origin, spec.cell)
    P = len(idx.coords)
    rng = np.random.default_rng(5)
    C = 64
    w = rng.normal(scale=0.3, size=(C, 9)).astype(np.float32)
    bias = rng.normal(scale=0.1, size=C).astype(np.float32)
    in_scale = float(np.abs(feats).max() / 127.0)
    if prec == "int8":
        ws_ = np.abs(w).max(axis=1) / 127.0
        wq = np.rint(w.astype(np.float64) / ws_[:, None]).clip(-128, 127)
        acc = np.einsum("pmj,cj->pmc", O.quantize(feats, in_scale).astype(np.float64), wq)
        alpha = (in_scale * ws_).astype(np.float32)
        y = (acc * alpha.astype(np.float64) + bias).astype(np.float32)
        wdev, adev = torch.from_numpy(wq.astype(np.int8)).cuda(), torch.from_numpy(alpha).cuda()
    else:
        y = (np.einsum("pmj,cj->pmc", feats.astype(np.float64), w.astype(np.float64)) + bias).astype(np.float32)
        wdev, adev = torch.from_numpy(w).cuda(), None
    y = np.where(mask[:, :, None], np.maximum(y, 0), -np.inf).max(axis=1)
    lib = N.load()
    g = pm.engine.GridSpec(grid=spec.grid, origin=spec.origin, cell=spec.cell, max_points=32, max_pillars=800).to_c()
    dpts = torch.from_numpy(pts).cuda()
    offs = torch.tensor([0, len(pts)], dtype=torch.int64, device="cuda")
    coords = torch.empty((1, 800, 2), dtype=torch.int32, device="cuda")
    counts = torch.empty((1, 800), dtype=torch.int32, device="cuda")
    pt_idx = torch.empty((1, 800, 32), dtype=torch.int32, device="cuda")
    npil = torch.empty((1,), dtype=torch.int32, device="cuda")
    wsb = lib.pmx_pillarize_workspace(ctypes.byref(g), 1, len(pts))
    wsp = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(lib.pmx_pillarize(dpts.data_ptr(), offs.data_ptr(), 1, len(pts), ctypes.byref(g), 800, coords.data_ptr(),
                              counts.data_ptr(), pt_idx.data_ptr(), npil.data_ptr(), wsp.data_ptr(), wsb,
                              N.stream_ptr()), "pillarize")
    d = N.PfnDesc(source=N.PMX_PFN_FROM_POINTS9, in_dtype=N.DTYPE_CODE[prec], n_features=9, channels=C,
                  max_points=32, relu=1, in_scale=in_scale if prec == "int8" else 0.0)
    bdev = torch.from_numpy(bias).cuda()
    for n_live in list(range(1, 71)) + [P - 1, P]:
        npil.fill_(n_live)
        rows = torch.full((800, C), -7.0, dtype=torch.float32, device="cuda")
        arr, n = N.outs_array([N.Out(ptr=rows.data_ptr(), scale=0.0, dtype=N.PMX_F32, c_stride=C, c_offset=0)])
        N.check(lib.pmx_pfn_pillars(ctypes.byref(d), ctypes.byref(g), 1, 800, dpts.data_ptr(), offs.data_ptr(), None,
                                    None, coords.data_ptr(), counts.data_ptr(), pt_idx.data_ptr(), npil.data_ptr(),
                                    wdev.data_ptr(), N.ptr(adev), bdev.data_ptr(), None, arr, n, None, None,
                                    N.stream_ptr()), "pfn_pillars")
        got = rows.cpu().numpy()
        np.testing.assert_allclose(got[:n_live], y[:n_live], rtol=1e-5, atol=1e-5, err_msg=str(n_live))
        assert (got[n_live:] == -7.0).all(), n_live
