"""Config-5 sensitivity sweep on the GPU: the K12 error reduction
against an f64 numpy sum, per-plan head errors against an independent engine run,
and the sweep's ranking / greedy candidates built from those errors."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import paper_2601_12638_b200 as pm

    return pm


@pytest.mark.parametrize("n", [0, 1, 1000, 3 * 2**20 + 7])
def test_sq_err_matches_f64(pm, n):
    import torch

    from paper_2601_12638_b200 import _native as N
    from paper_2601_12638_b200.sweep import _sq_err, sq_err_workspace

    lib = N.require_cuda()
    rng = np.random.default_rng(n)
    a = rng.normal(size=n).astype(np.float32)
    b = (a + rng.normal(scale=0.01, size=n)).astype(np.float32)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    ws = sq_err_workspace(lib)
    _sq_err(lib, ta, tb, acc, ws)
    _sq_err(lib, ta, tb, acc, ws)  # accumulates
    got = acc.cpu().numpy()
    want = 2 * np.array([np.sum((a.astype(np.float64) - b) ** 2), np.sum(b.astype(np.float64) ** 2)])
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
    acc2 = torch.zeros(2, dtype=torch.float64, device="cuda")
    _sq_err(lib, ta, tb, acc2, ws)
    _sq_err(lib, ta, tb, acc2, ws)
    assert acc2.cpu().numpy().tobytes() == got.tobytes()  # deterministic


def test_small_sweep(pm):
    import torch

    from paper_2601_12638_b200 import sweep as S

    cfg = pm.PointPillarsConfig.small()
    graph = pm.build_pointpillars(cfg, seed=3)
    calib = [pm.make_frame(4000, 50 + i, cfg, 0.01) for i in range(2)]
    stats = pm.calibrate_frames(graph, calib, cfg)
    frames = [pm.make_frame(3000 + 500 * i, 200 + i, cfg) for i in range(3)]
    res = S.sensitivity_sweep(graph, stats, frames, cfg, batch=2, k=3)
    errs = res["layer_errors"]
    assert sorted(errs) == [l.index for l in graph.weight_layers]
    assert all(np.isfinite(e) and e > 0 for e in errs.values())
    assert res["ranking"] == S.select_topk(errs, len(errs))
    assert list(res["candidates"]) == [c.label() for c in S.greedy_candidates(res["ranking"], 3)]

    # independent check of two plans: batch-1 engines, host-side f64 error
    def heads(plan):
        out = []
        for f in frames:
            eng = pm.PointPillarsEngine(graph, plan, stats, cfg, batch=1, max_points_per_frame=len(f))
            eng.load_points([f])
            eng.run()
            torch.cuda.synchronize()
            out.append(eng.cg.heads_cat[0].double().cpu().numpy())
        return np.stack(out)

    ref = heads(pm.PrecisionPlan())
    for idx in (res["ranking"][0], res["ranking"][-1]):
        y = heads(pm.PrecisionPlan(default=pm.DType.FP32, overrides={idx: pm.DType.INT8}))
        want = np.sqrt(np.sum((y - ref) ** 2) / np.sum(ref ** 2))
        assert errs[idx] == pytest.approx(want, rel=1e-9)
    lab = next(iter(res["candidates"]))
    y = heads(pm.parse_plan_label(lab))
    assert res["candidates"][lab] == pytest.approx(np.sqrt(np.sum((y - ref) ** 2) / np.sum(ref ** 2)), rel=1e-9)
