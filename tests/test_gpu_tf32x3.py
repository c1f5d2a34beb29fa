"""FP32 layers on the tensor cores (3xTF32, PMX_F32X2): the (hi, lo) activation split is
exact, every KITTI layer class matches the f64 oracle within the T1 bar (1e-5 rel L2; the
tensor core truncates while accumulating, so 3xTF32 sits at ~1e-6..1e-5 where the SIMT
FFMA kernel is at ~3e-7), the SIMT FP32 kernel agrees, and the engine routes FP32 plans
(not calibration, which keeps exact f32 FMA) through the tcgen05 path."""

import ctypes

import numpy as np
import pytest

from oracle import pillars_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_f32x2_split_is_exact(pm):
    import torch

    from paper_2601_12638_b200 import _native as N
    from paper_2601_12638_b200.engine import tf32_split

    lib = N.load()
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(scale=s, size=4096) for s in (1e-30, 1e-3, 1.0, 1e4, 1e30)]).astype(np.float32)
    x = np.concatenate([x, np.array([0.0, -0.0, 1.0, -1.0, 3.4e38, -3.4e38, 1e-45, np.inf, -np.inf], np.float32)])
    C = 16
    x = np.concatenate([x, np.zeros((-len(x)) % C, np.float32)])
    pix = len(x) // C
    out = torch.full((pix, 2 * C), 7.0, dtype=torch.float32, device="cuda")
    arr, n = N.outs_array([N.Out(ptr=out.data_ptr(), scale=0.0, dtype=N.PMX_F32X2, c_stride=2 * C, c_offset=0)])
    N.check(lib.pmx_cast_out(torch.from_numpy(x).cuda().data_ptr(), pix, C, arr, n, None, N.stream_ptr()), "cast")
    o = out.cpu().numpy().reshape(pix, 2, C)
    hi, lo = o[:, 0].reshape(-1), o[:, 1].reshape(-1)
    fin = np.isfinite(x)
    np.testing.assert_array_equal(hi[fin] + lo[fin], x[fin])  # hi + lo == x exactly (f32 add)
    assert not (hi[fin].view(np.uint32) & 0x1FFF).any()        # hi is a TF32 value
    hh, ll = tf32_split(x)                                      # the host twin used for weights
    np.testing.assert_array_equal(hh, hi)
    np.testing.assert_array_equal(ll[fin], lo[fin])
    np.testing.assert_array_equal(hi[~fin], x[~fin])


SHAPES = {  # cin, cout, k, stride, (h, w), kind
    "conv_s2": (64, 64, 3, 2, (62, 54), "conv2d"),
    "conv_s1_64": (64, 64, 3, 1, (31, 27), "conv2d"),
    "conv_s1_256": (256, 256, 3, 1, (16, 14), "conv2d"),
    "conv_s2_128": (128, 256, 3, 2, (32, 28), "conv2d"),
    "deconv1": (64, 128, 1, 1, (31, 27), "deconv2d"),
    "deconv2": (128, 128, 2, 2, (16, 14), "deconv2d"),
    "deconv4": (256, 128, 4, 4, (8, 7), "deconv2d"),
    "head": (384, 20, 1, 1, (31, 27), "conv2d"),
}


@pytest.mark.parametrize("name", list(SHAPES))
def test_tf32x3_layer_vs_f64_oracle_and_simt(pm, name):
    from paper_2601_12638_b200 import _native as N
    from paper_2601_12638_b200 import engine as E

    cin, cout, k, s, hw, kind = SHAPES[name]
    rng = np.random.default_rng(hash(name) % 2**32)
    x = np.maximum(rng.normal(size=(2, cin) + hw), 0).astype(np.float32)
    w = rng.normal(scale=np.sqrt(2.0 / (cin * k * k)), size=(cout, cin, k, k)).astype(np.float32)
    b = rng.normal(scale=0.1, size=cout).astype(np.float32)
    deconv = kind == "deconv2d"
    pad = (0, 0) if (deconv or k == 1) else (1, 1)
    layer = pm.LayerSpec(name="l", kind=kind, index=1, weight=w, bias=b, relu=name != "head",
                         conv=pm.ConvParams(stride=(s, s), padding=pad))
    graph = pm.ModelGraph(layers=(layer,))
    cg = E.CompiledGraph(graph, None, source="array", in_shape=x.shape)
    assert cg.x3 == {"l"}  # the FP32 layer runs on the 3xTF32 tensor-core kernel
    got = pm.forward(graph, x)
    with O.accumulate_in(np.float64):
        want = O.run_weight_layer(layer, x, None)
    err = rel_l2(got, want)
    lib = N.load()
    lib.pmx_set_conv_backend(1)
    try:
        simt = pm.forward(graph, x)
    finally:
        lib.pmx_set_conv_backend(0)
    print(name, "3xTF32 vs f64", err, "SIMT vs f64", rel_l2(simt, want))
    assert err <= 1e-5  # SURVEY §8(d) T1 bar for a layer
    assert rel_l2(got, simt) <= 1e-5


def test_fp32_plan_full_size_on_tensor_cores(pm):
    """Every conv / deconv / head of the FP32 plan takes the 3xTF32 path at KITTI size and
    the heads stay within the FP32 bar (1e-4) of the f32 oracle."""
    cfg = pm.PointPillarsConfig()
    graph = pm.build_pointpillars(cfg, seed=0)
    frame = pm.make_frame(20000, 1, cfg)
    eng = pm.PointPillarsEngine(graph, "FP32", None, cfg, batch=1, max_points_per_frame=20000)
    convs = {l.name for l in graph.weight_layers if l.index != 1}
    assert eng.cg.x3 == convs
    eng.load_points([frame])
    eng.run()
    heads = {k: v.cpu().numpy() for k, v in eng.heads_nchw().items()}
    planned = pm.apply_plan(pm.fold_all_bn(graph), pm.PrecisionPlan())
    sample, _ = O.pillarize_kitti(frame, cfg.grid_spec())
    want = O.forward(O.folded_graph(planned, {l.index: "fp32" for l in planned.weight_layers}), sample)
    for name, ref in zip(pm.pointpillars.HEADS, want):
        e = rel_l2(heads[name][0], ref[0])
        print(name, e)
        assert e <= 1e-4, name
