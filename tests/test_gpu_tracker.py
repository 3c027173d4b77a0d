"""GPU oracle tracker (scene.oracle_tracks, K2 "dominant" mode) against the reference's own
oracle_track (scene.py:166-240).

Fixtures: tracker_kats.npz (the scenes of the reference's tests/test_scene.py:67-156: dominant
images, static-scene identity tracks, coverage = valid, keyed noise, pure translation) and the
TRKF tracks of scene21 / scene7 / cfg1, all produced by the reference in the build container.
Contract: dominant gid image and depth image bit-exact; valid mask bit-exact; targets within the
float32 rounding of the TRKF layout the GPU path emits (one float32 ulp: the device transport's
matrix products may round the last float64 bit differently from numpy's BLAS).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2604_02586_b200.scene import generate_scene, oracle_tracks  # noqa: E402
from tests import golden_data as gd  # noqa: E402


def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _assert_f32_close(got, ref, valid):
    g = got[valid].astype(np.float32)
    r = ref[valid].astype(np.float32)
    ulp = np.spacing(np.abs(r))
    bad = np.abs(g.astype(np.float64) - r.astype(np.float64)) > ulp
    assert not bad.any(), f"{int(bad.sum())} targets beyond one float32 ulp"
    return float(np.mean(g == r)) if g.size else 1.0


@pytest.mark.parametrize("tag", sorted(gd.TRACKER_SCENES))
def test_dominant_and_tracks_vs_reference(tag):
    _need_cuda()
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load("tracker_kats")
    meta, views = gd.tracker_case(d, tag)
    args, kw = gd.TRACKER_SCENES[tag]
    scene = generate_scene(*args, **kw)
    eng = FrameEngine().bin(scene.frames[0], scene.cameras)
    vs = sorted(views)
    tgt, val = oracle_tracks(scene, meta["frame"], noise_sigma_px=meta["noise"], seed=meta["seed"],
                             engine=eng, views=vs)
    tgt, val = tgt.cpu().numpy(), val.cpu().numpy().astype(bool)
    for k, v in enumerate(vs):
        ref = views[v]
        gid, dep = eng.dominant_gaussians(v)
        np.testing.assert_array_equal(gid.cpu().numpy(), ref["gid"])
        np.testing.assert_array_equal(dep.cpu().numpy(), ref["depth"])
        np.testing.assert_array_equal(val[k], ref["valid"])
        _assert_f32_close(tgt[k], ref["target"], ref["valid"])


@pytest.mark.parametrize("name", sorted(gd.SCENE_TRACKS))
def test_tracks_vs_reference_trkf(name):
    _need_cuda()
    d = gd.load(name)
    tgt_ref, val_ref = gd.tracks(d)
    args, kw, sigma = gd.SCENE_TRACKS[name]
    scene = generate_scene(*args, **kw)
    tgt, val = oracle_tracks(scene, 1, noise_sigma_px=sigma, seed=0)
    tgt, val = tgt.cpu().numpy(), val.cpu().numpy().astype(bool)
    np.testing.assert_array_equal(val, val_ref)
    exact = _assert_f32_close(tgt, tgt_ref, val_ref)
    print(f"{name}: {exact:.4%} of valid targets bit-identical to the reference's TRKF tracks")
