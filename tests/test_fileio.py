"""On-disk formats (fileio.py of the reference): byte-identical writers, exact round trips, both
directions against the reference package when it is importable, and MalformedFile on the
malformed inputs the reference rejects (tests/test_fileio.py of the reference)."""

import os
import struct
import sys

import numpy as np
import pytest

from paper_2604_02586_b200 import fileio
from paper_2604_02586_b200.errors import MalformedFile
from paper_2604_02586_b200.motion2d import TrackField
from paper_2604_02586_b200.scene import generate_scene

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref_fileio():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF)
    try:
        import gausstrack.fileio as rf
        return rf
    finally:
        sys.path.remove(REF)


@pytest.fixture(scope="module")
def scene():
    return generate_scene(3, 40, 3, 3, width=64, height=48, focal=60)


def _tf(seed=0, w=7, h=5, view=2):
    rng = np.random.default_rng(seed)
    tgt = rng.normal(0, 30, (h, w, 2)).astype(np.float32).astype(np.float64)
    val = rng.random((h, w)) < 0.7
    tgt[~val] = np.nan
    return TrackField(view, w, h, tgt, val)


def _read(p):
    with open(p, "rb") as fh:
        return fh.read()


def test_gaussians_round_trip(tmp_path, scene):
    p = tmp_path / "g.txt"
    fileio.save_gaussians(p, scene.frames[1])
    rows = fileio.load_gaussian_rows(p)
    np.testing.assert_array_equal(rows[:, [0, 1, 2, 7, 8, 9, 10]],
                                  scene.frames[1][:, [0, 1, 2, 7, 8, 9, 10]])
    np.testing.assert_allclose(rows[:, 3:7], scene.frames[1][:, 3:7], rtol=0, atol=1e-15)
    g = fileio.load_gaussians(p)
    assert len(g) == 40 and np.array_equal(g[5].mean, rows[5, 0:3])


def test_gaussians_match_reference(tmp_path, scene, ref_fileio):
    ours, theirs = tmp_path / "a.txt", tmp_path / "b.txt"
    gl = scene.gaussians(2)          # Gaussian3D objects (quaternions renormalised)
    fileio.save_gaussians(ours, gl)
    ref_fileio.save_gaussians(theirs, gl)
    assert _read(ours) == _read(theirs)
    ref = ref_fileio.load_gaussians(ours)
    rows = fileio.load_gaussian_rows(theirs)
    for r, g in zip(rows, ref):
        assert np.array_equal(r, np.concatenate([g.mean, g.rotation, g.scale, [g.opacity]]))


def test_cameras_match_reference(tmp_path, scene, ref_fileio):
    ours, theirs = tmp_path / "a.txt", tmp_path / "b.txt"
    fileio.save_cameras(ours, scene.cameras)
    ref_fileio.save_cameras(theirs, scene.cameras)
    assert _read(ours) == _read(theirs)
    for a, b in zip(fileio.load_cameras(theirs), ref_fileio.load_cameras(ours)):
        assert np.array_equal(a.as_row(), np.concatenate(
            [b.rotation.ravel(), b.translation, [b.fx, b.fy, b.cx, b.cy, b.width, b.height]]))


@pytest.mark.parametrize("kind", ["text", "binary"])
def test_trackfield_match_reference(tmp_path, ref_fileio, kind):
    tf = _tf()
    ours, theirs = tmp_path / "a", tmp_path / "b"
    getattr(fileio, f"save_trackfield_{kind}")(ours, tf)
    getattr(ref_fileio, f"save_trackfield_{kind}")(theirs, tf)
    assert _read(ours) == _read(theirs)
    a = getattr(fileio, f"load_trackfield_{kind}")(theirs)
    b = getattr(ref_fileio, f"load_trackfield_{kind}")(ours)
    assert (a.view_id, a.width, a.height) == (b.view_id, b.width, b.height)
    np.testing.assert_array_equal(a.valid, b.valid)
    np.testing.assert_array_equal(a.target[a.valid], b.target[b.valid])


def test_trkf_batch_layout(tmp_path):
    tfs = [_tf(seed=s, view=v) for s, v in ((1, 0), (2, 1), (3, 4))]
    paths = []
    for tf in tfs:
        paths.append(tmp_path / fileio.track_filename(tf.view_id, 1))
        fileio.save_trackfield_binary(paths[-1], tf)
    tgt, val, ids = fileio.load_trkf_batch(paths, pinned=False)
    assert ids == [0, 1, 4]
    assert tuple(tgt.shape) == (3, 5, 7, 2) and tgt.dtype.itemsize == 4
    for v, tf in enumerate(tfs):
        np.testing.assert_array_equal(val[v].numpy() != 0, tf.valid)
        np.testing.assert_array_equal(tgt[v].numpy()[tf.valid], tf.target[tf.valid])
    # the device-layout writer produces the same bytes
    p2 = tmp_path / "again.trk"
    fileio.save_trkf_arrays(p2, 0, tgt[0].numpy(), val[0].numpy())
    assert _read(p2) == _read(paths[0])


def test_trkf_batch_rejects_mixed_sizes(tmp_path):
    a, b = tmp_path / "a.trk", tmp_path / "b.trk"
    fileio.save_trackfield_binary(a, _tf(w=7, h=5))
    fileio.save_trackfield_binary(b, _tf(w=6, h=5))
    with pytest.raises(MalformedFile):
        fileio.load_trkf_batch([a, b], pinned=False)


def test_malformed_inputs(tmp_path, scene):
    bad = tmp_path / "bad"
    cases = {
        "load_gaussians": ["GAUSS3D v2 1\n", "GAUSS3D v1 2\n" + "1 " * 11 + "\n",
                           "GAUSS3D v1 1\n1 2 3\n",
                           "GAUSS3D v1 1\n0 0 0 1 0 0 0 1 -1 1 0.5\n",
                           "GAUSS3D v1 1\n0 0 0 1 0 0 0 1 1 1 1.5\n"],
        "load_cameras": ["CAMERA v2\n", "CAMERA v1\n1 2 3\n"],
        "load_trackfield_text": ["TRACKFIELD v1 0 2 2\n1 2 1\n"],
    }
    for fn, texts in cases.items():
        for text in texts:
            bad.write_text(text)
            with pytest.raises(MalformedFile):
                getattr(fileio, fn)(bad)
    good = tmp_path / "good.trk"
    fileio.save_trackfield_binary(good, _tf())
    raw = _read(good)
    for blob in (b"TRKX" + raw[4:], raw[:10], raw[:16 + 20], raw[:-3]):
        bad.write_bytes(blob)
        with pytest.raises(MalformedFile):
            fileio.load_trackfield_binary(bad)
        with pytest.raises(MalformedFile):
            fileio.load_trkf_batch([bad], pinned=False)
    with pytest.raises(MalformedFile):
        fileio.load_gaussians(tmp_path / "missing.txt")
    assert struct.unpack("<III", raw[4:16]) == (2, 7, 5)


def test_scene_dir_round_trip(tmp_path, scene):
    d = tmp_path / "scene"
    fileio.save_scene(d, scene)
    back = fileio.load_scene(d)
    assert back.n_frames == 3 and back.n_gaussians == 40
    for a, b in zip(back.frames, scene.frames):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-15)
    with pytest.raises(MalformedFile):
        fileio.load_scene(tmp_path)


def test_scene_dir_readable_by_reference(tmp_path, scene, ref_fileio):
    d = tmp_path / "scene"
    fileio.save_scene(d, scene)
    ref = ref_fileio.load_scene(str(d))
    assert ref.n_frames == 3
    ours = fileio.load_scene(d)
    for t in range(3):
        for r, g in zip(ours.frames[t], ref.frames[t]):
            assert np.array_equal(r, np.concatenate([g.mean, g.rotation, g.scale, [g.opacity]]))
