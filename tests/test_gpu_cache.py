"""Clip contribution cache (ts_frame_cache): K2 runs once per binning without tracks; every target
frame then applies its tracks to the cached contributions (the GPU form of the reference's frame-0
weight-map reuse across a clip, pipeline.py:191-196).  The cached path must give what the
per-frame rasterization gives: integer counts bit-exact, sums to rounding (another summation
order), statuses and updates to the SURVEY §8(c) tolerances, for several target frames of one
clip, against the uncached path and against the CPU oracle."""

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


def _tracks(target, valid, shift):
    t = (target + np.array([shift, -0.5 * shift])).astype(np.float32)
    return t, valid.astype(np.uint8)


def _compare(a, b, n, nv):
    for k in ("pixel_count", "static_pixel_count"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    for k in ("weight_sum", "static_weight_sum"):
        x, y = getattr(a, k).cpu().numpy(), getattr(b, k).cpu().numpy()
        np.testing.assert_allclose(x, y, rtol=1e-12, atol=1e-300, err_msg=k)
    sa, sb = a.motion_status.cpu().numpy(), b.motion_status.cpu().numpy()
    assert (sa != sb).sum() <= max(1, 1e-5 * n * nv)  # threshold ties under another sum order
    st = (sa == 1) & (sb == 1)
    ma, mb = a.motion_a.cpu().numpy()[st], b.motion_a.cpu().numpy()[st]
    assert np.sum(np.abs(ma - mb).max(axis=(1, 2)) > 1e-8) <= max(1, 1e-5 * st.sum())
    ua, ub = a.status.cpu().numpy(), b.status.cpu().numpy()
    assert (ua != ub).sum() <= max(1, 1e-4 * n)
    u = (ua == 1) & (ub == 1)
    da, db = a.delta_mean.cpu().numpy()[u], b.delta_mean.cpu().numpy()[u]
    assert np.sum(np.abs(da - db).max(axis=1) > 1e-9) <= max(1, 1e-4 * u.sum())


@pytest.mark.parametrize("scene", ["scene7", "cfg1"])
def test_cache_matches_per_frame_raster(scene):
    _need_cuda()
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load(scene)
    target, valid = gd.tracks(d)
    g, cams = d["gaussians"], d["cameras"]
    n, nv = len(g), len(cams)
    plain = FrameEngine().bin(g, cams)
    cached = FrameEngine().bin(g, cams).build_cache()
    for shift in (0.0, 0.6, -1.3):  # three target frames of one clip
        t, v = _tracks(target, valid, shift)
        a = plain.compensate(t, v)
        b = cached.compensate(t, v)
        torch.cuda.synchronize()
        _compare(a, b, n, nv)
    # the oracle on the last frame
    upd, mots, accs = oracle.compensate(g, cams, list(t.astype(np.float64)), list(v.astype(bool)))
    np.testing.assert_array_equal(b.pixel_count.cpu().numpy().reshape(nv, n),
                                  np.stack([x["pixel_count"] for x in accs]))
    _check_updates(b.status.cpu().numpy(), b.delta_mean.cpu().numpy(), b.rotation.cpu().numpy(),
                   b.scale.cpu().numpy(), upd["status"], upd["delta_mean"], upd["rotation"],
                   upd["scale"], g)
    # a new binning invalidates the cache; dropping it returns to the per-frame raster
    cached.drop_cache()
    c = cached.compensate(t, v)
    torch.cuda.synchronize()
    _compare(a, c, n, nv)


def test_cache_at_scale_cfg3():
    """BASELINE configs[2] (200k x 27 views): cached vs per-frame K2, two target frames."""
    _need_cuda()
    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.scene import generate_scene, oracle_tracks
    scene = generate_scene(0, 200_000, 27, 7, focal=520, width=640, height=360,
                           translate_mag=0.12, rotate_deg=3.0)
    eng = FrameEngine().bin(scene.frames[0], scene.cameras)
    n, nv = len(scene.frames[0]), len(scene.cameras)
    outs = {}
    for f in (3, 6):
        tgt, val = oracle_tracks(scene, f, engine=eng)
        outs[f] = (tgt, val, eng.compensate(tgt, val))
    eng.build_cache()
    for f, (tgt, val, ref) in outs.items():
        got = eng.compensate(tgt, val)
        torch.cuda.synchronize()
        _compare(ref, got, n, nv)


@pytest.mark.parametrize("use_cache", [False, True])
def test_compact_fits_same_updates(use_cache):
    """motions=False: K3 keeps its fits compact (cache / touched list) and K4 reads them in place
    (only the statuses are written densely) -- the updates must equal the dense path's bit for
    bit, since K4 reads the same numbers."""
    _need_cuda()
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load("scene21")
    target, valid = gd.tracks(d)
    eng = FrameEngine().bin(d["gaussians"], d["cameras"])
    if use_cache:
        eng.build_cache()
    t, v = _tracks(target, valid, 0.4)
    a = eng.compensate(t, v)
    b = eng.compensate(t, v, motions=False)
    torch.cuda.synchronize()
    assert b.motion_status is None
    for k in ("delta_mean", "rotation", "scale", "status"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k


def test_cache_long_runs_and_f64_tracks():
    """Large Gaussians (runs of far more than 128 cached contributions: the chunked per-frame
    kernel's scratch reduction, k23_cached_multi) and float64 tracks (the double instantiation):
    cached == per-frame to rounding, and the oracle's counts exactly."""
    _need_cuda()
    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.scene import generate_scene, oracle_tracks
    scene = generate_scene(3, 400, 6, 3, focal=300, width=320, height=240,
                           scale_range=(0.03, 0.12))
    g, cams = scene.frames[0], scene.cameras
    n, nv = len(g), len(cams)
    plain = FrameEngine().bin(g, cams)
    cached = FrameEngine().bin(g, cams).build_cache()
    nrec, nw = cached.cache_info()
    assert nrec > 0 and nw > 0
    tgt, val = oracle_tracks(scene, 2, engine=plain)
    tgt64 = tgt.to(torch.float64)
    for t in (tgt, tgt64):
        a = plain.compensate(t, val)
        b = cached.compensate(t, val)
        torch.cuda.synchronize()
        _compare(a, b, n, nv)
    # some gv has a run longer than one 128-contribution chunk
    assert int(b.pixel_count.max()) > 128
    rows = np.array([c.as_row() for c in cams])
    upd, mots, accs = oracle.compensate(g, rows, list(tgt64.cpu().numpy()),
                                        list(val.cpu().numpy().astype(bool)))
    np.testing.assert_array_equal(b.pixel_count.cpu().numpy().reshape(nv, n),
                                  np.stack([x["pixel_count"] for x in accs]))


def test_cache_grouped_rig():
    """Mixed image sizes (one plan per same-size group): every plan builds its cache."""
    _need_cuda()
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    g = d["gaussians"]
    cams = d["cameras"].copy()
    targets, valids = [], []
    for v in range(len(cams)):
        if 3 <= v <= 5:
            cams[v, 16], cams[v, 17] = 800, 500
            targets.append(np.ascontiguousarray(target[v, :500, :800]).astype(np.float32))
            valids.append(np.ascontiguousarray(valid[v, :500, :800]).astype(np.uint8))
        else:
            targets.append(target[v].astype(np.float32))
            valids.append(valid[v].astype(np.uint8))
    plain = FrameEngine().bin(g, cams)
    cached = FrameEngine().bin(g, cams).build_cache()
    assert cached.grouped
    a = plain.compensate(targets, valids)
    b = cached.compensate(targets, valids)
    c = cached.compensate(targets, valids, motions=False)
    torch.cuda.synchronize()
    _compare(a, b, len(g), len(cams))
    for k in ("delta_mean", "rotation", "scale", "status"):
        assert torch.equal(getattr(b, k), getattr(c, k)), k
