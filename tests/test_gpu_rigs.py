"""Camera rigs beyond one binning plan: views of different image sizes (the reference rasterizes
each view at its own size, pipeline.py:117-120; accumulate_view checks sizes per view,
motion2d.py:132-135) and more than 64 views.  FrameEngine bins same-size groups of <= 64 views on
separate plans (K1-K3 each) and fuses all views in one K4 (ts_update_all); results are checked
against the CPU oracle run view by view: counts bit-exact, statuses and updates to SURVEY §8(c)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from tests import golden_data as gd  # noqa: E402
from tests.test_gpu_parity import _check_updates  # noqa: E402


def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _check_vs_oracle(g, cams, targets, valids, out):
    n, nv = len(g), len(cams)
    upd, mots, accs = oracle.compensate(g, cams, [t.astype(np.float64) for t in targets],
                                        [v.astype(bool) for v in valids])
    np.testing.assert_array_equal(out.pixel_count.cpu().numpy().reshape(nv, n),
                                  np.stack([a["pixel_count"] for a in accs]))
    np.testing.assert_allclose(out.weight_sum.cpu().numpy().reshape(nv, n),
                               np.stack([a["weight_sum"] for a in accs]), rtol=1e-9, atol=1e-300)
    ms = out.motion_status.cpu().numpy().reshape(nv, n)
    assert (ms != np.stack([m["status"] for m in mots])).sum() <= max(1, 1e-4 * n * nv)
    _check_updates(out.status.cpu().numpy(), out.delta_mean.cpu().numpy(),
                   out.rotation.cpu().numpy(), out.scale.cpu().numpy(), upd["status"],
                   upd["delta_mean"], upd["rotation"], upd["scale"], g)
    return upd


def test_mixed_image_sizes():
    _need_cuda()
    from paper_2604_02586_b200 import Config, compensate_frame
    from paper_2604_02586_b200.core import camera_from_row, gaussians_from_array
    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.motion2d import TrackField
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    g = d["gaussians"]
    cams = d["cameras"].copy()
    # views 3..5 see an 800x500 window of the same image plane (same intrinsics)
    targets, valids = [], []
    for v in range(len(cams)):
        if 3 <= v <= 5:
            cams[v, 16], cams[v, 17] = 800, 500
            targets.append(np.ascontiguousarray(target[v, :500, :800]).astype(np.float32))
            valids.append(np.ascontiguousarray(valid[v, :500, :800]).astype(np.uint8))
        else:
            targets.append(target[v].astype(np.float32))
            valids.append(valid[v].astype(np.uint8))
    eng = FrameEngine().bin(g, cams)
    assert eng.grouped and len(eng._groups) == 3
    out = eng.compensate(targets, valids)
    torch.cuda.synchronize()
    upd = _check_vs_oracle(g, cams, targets, valids, out)
    # the public entry point with per-view TrackFields of different sizes
    frame1 = gaussians_from_array(g)
    tfs = [TrackField(v, int(cams[v, 16]), int(cams[v, 17]), targets[v].astype(np.float64),
                      valids[v].astype(bool)) for v in range(len(cams))]
    res = compensate_frame(frame1, [camera_from_row(c) for c in cams], tfs, Config(),
                           frame_index=1, regularize=False)
    assert res.tallies["solved"] == int((out.status.cpu().numpy() == 1).sum())
    assert abs(res.tallies["solved"] - int(upd["status"].sum())) <= 2


def test_more_than_64_views():
    _need_cuda()
    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.scene import generate_scene
    scene = generate_scene(5, 600, 70, 2, width=320, height=240, focal=260)
    cams = np.array([c.as_row() for c in scene.cameras])
    targets, valids = [], []
    rel = oracle.relative_rotations(scene.frames[0], scene.frames[1])
    for v in range(len(cams)):
        wm = oracle.rasterize(scene.frames[0], cams[v])
        t, va = oracle.oracle_track(scene.frames[0], scene.frames[1], cams[v], wm, v, 1, rel=rel)
        targets.append(t.astype(np.float32))
        valids.append(va.astype(np.uint8))
    eng = FrameEngine().bin(scene.frames[0], cams)
    assert eng.grouped and [(a, b) for a, b, _ in eng._groups] == [(0, 64), (64, 70)]
    out = eng.compensate(targets, valids)
    torch.cuda.synchronize()
    upd = _check_vs_oracle(scene.frames[0], cams, targets, valids, out)
    # Gaussians seen by views on both sides of the 64-view boundary were fused
    ms = out.motion_status.cpu().numpy().reshape(70, -1)
    both = (ms[:64] == 1).any(0) & (ms[64:] == 1).any(0) & (upd["status"] == 1)
    assert both.sum() > 10
