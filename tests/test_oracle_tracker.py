"""Pin the CPU oracle tracker and the grouped update_all (oracle/) against the reference.

CPU only.  `oracle.dominant_gaussians` / `oracle.oracle_track` restate scene.py:166-240; they
produce the CPU arm's inputs in bench.py (no repo library involved) and check the GPU tracker.
The fixtures come from the reference itself (tests/golden/make_golden.py: tracker_kats and the
scene fixtures' TRKF tracks); the tracker cases are the scenes of the reference's
tests/test_scene.py:67-156.
"""

import numpy as np
import pytest

import oracle
from paper_2604_02586_b200.scene import generate_scene
from tests import golden_data as gd


@pytest.mark.parametrize("tag", sorted(gd.TRACKER_SCENES))
def test_tracker_kats(tag):
    d = gd.load("tracker_kats")
    meta, views = gd.tracker_case(d, tag)
    args, kw = gd.TRACKER_SCENES[tag]
    scene = generate_scene(*args, **kw)
    np.testing.assert_array_equal(scene.frames[0], meta["g0"])
    np.testing.assert_array_equal(scene.frames[meta["frame"]], meta["g1"])
    for v, ref in views.items():
        cam = meta["cameras"][v]
        wm = oracle.rasterize(scene.frames[0], cam)
        gid, dep = oracle.dominant_gaussians(wm, int(cam[16]), int(cam[17]))
        np.testing.assert_array_equal(gid, ref["gid"])
        np.testing.assert_array_equal(dep, ref["depth"])
        tgt, val = oracle.oracle_track(scene.frames[0], scene.frames[meta["frame"]], cam, wm, v,
                                       meta["frame"], meta["noise"], meta["seed"])
        np.testing.assert_array_equal(val, ref["valid"])
        np.testing.assert_array_equal(tgt, ref["target"])


@pytest.mark.parametrize("name", sorted(gd.SCENE_TRACKS))
def test_tracks_match_reference_trkf(name):
    """The TRKF-rounded tracks of the scene fixtures, bit-exact (valid mask and targets)."""
    d = gd.load(name)
    tgt_ref, val_ref = gd.tracks(d)
    args, kw, sigma = gd.SCENE_TRACKS[name]
    scene = generate_scene(*args, **kw)
    rel = oracle.relative_rotations(scene.frames[0], scene.frames[1])
    for v, cam in enumerate(d["cameras"]):
        wm = oracle.rasterize(scene.frames[0], cam)
        tgt, val = oracle.oracle_track(scene.frames[0], scene.frames[1], cam, wm, v, 1, sigma,
                                       rel=rel)
        np.testing.assert_array_equal(val, val_ref[v])
        np.testing.assert_array_equal(tgt.astype("<f4").astype(np.float64)[val], tgt_ref[v][val])


def test_dominant_ties_by_smaller_gid():
    """scene.py:178: equal alpha*T at a pixel -> the smaller gaussian id wins."""
    wm = dict(pixel_x=np.array([1, 1, 1, 0], np.int32), pixel_y=np.array([0, 0, 0, 0], np.int32),
              gaussian_id=np.array([7, 3, 5, 9], np.int64),
              alpha=np.array([0.5, 0.25, 0.5, 0.1]), transmittance=np.array([0.5, 1.0, 0.5, 1.0]),
              depth=np.array([3.0, 1.0, 2.0, 4.0]))
    gid, dep = oracle.dominant_gaussians(wm, 2, 1)
    assert gid.tolist() == [[9, 3]] and dep.tolist() == [[4.0, 1.0]]


@pytest.mark.parametrize("name", ["scene21", "scene7", "cfg1"])
def test_grouped_update_all_equals_loop(name):
    """The grouped LAPACK calls of oracle.update_all give the reference loop's bits."""
    d = gd.load(name)
    mot = gd.motions(d)
    a = oracle.update_all(d["gaussians"], mot, d["cameras"])
    b = oracle.update_all(d["gaussians"], mot, d["cameras"], loop=True)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
