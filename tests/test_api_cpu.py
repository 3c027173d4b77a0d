"""Host-side API of the drop-in package (no GPU needed): types, validation, config, clips, lazy
lists and the scene generator, mirroring the reference's own unit tests (tests/test_core.py,
test_fileio.py config parsing, test_pipeline.py clip protocol, test_scene.py determinism)."""

import numpy as np
import pytest

import paper_2604_02586_b200 as p
from paper_2604_02586_b200 import errors
from paper_2604_02586_b200.core import (camera_from_row, cameras_array, gaussians_array,
                                        gaussians_from_array)
from paper_2604_02586_b200.motion2d import MotionAccumulator, ViewMotionList, accumulate
from paper_2604_02586_b200.multiview import MotionUpdateList
from paper_2604_02586_b200.pipeline import GaussianList, apply_update_rows
from paper_2604_02586_b200.scene import generate_scene
from tests import golden_data as gd


def test_public_names_match_reference_hot_path():
    for name in ["Gaussian3D", "CameraView", "TrackField", "Config", "rasterize_weights",
                 "accumulate_view", "solve_view", "solve_all_views", "update_all",
                 "compensate_frame", "WeightMap", "Status", "MotionUpdate", "ViewMotion",
                 "triangulate_mean", "solve_covariance3d", "decompose_covariance",
                 "update_gaussian", "accumulate", "solve_motion", "segment_clips",
                 "FrameResult", "invert_2x2", "Sym3", "AffineMotion", "Gaussian2D"]:
        assert hasattr(p, name), name


def test_gaussian_validation_and_normalisation():
    g = p.Gaussian3D([1, 2, 3], [2, 0, 0, 0], [0.1, 0.2, 0.3], 0.5)
    np.testing.assert_array_equal(g.rotation, [1, 0, 0, 0])
    with pytest.raises(ValueError):
        p.Gaussian3D([0, 0, 0], [1, 0, 0, 0], [0.1, -0.2, 0.3], 0.5)
    with pytest.raises(ValueError):
        p.Gaussian3D([0, 0, 0], [1, 0, 0, 0], [0.1, 0.2, 0.3], 0.0)
    with pytest.raises(ValueError):
        p.Gaussian3D([0, 0, 0], [0, 0, 0, 0], [0.1, 0.2, 0.3], 0.5)


def test_camera_validation():
    with pytest.raises(ValueError):
        p.CameraView(np.diag([1.0, 1.0, -1.0]), np.zeros(3), 1, 1, 0, 0, 4, 4)
    with pytest.raises(ValueError):
        p.CameraView(2 * np.eye(3), np.zeros(3), 1, 1, 0, 0, 4, 4)
    cam = p.CameraView(np.eye(3), [0, 0, 1], 100, 90, 32, 24, 64, 48)
    np.testing.assert_array_equal(camera_from_row(cam.as_row()).rotation, cam.rotation)
    assert cam.projection_matrix().shape == (3, 4)


def test_projection_helpers():
    cam = p.CameraView(np.eye(3), np.zeros(3), 100, 100, 32, 24, 64, 48)
    m, z = p.project_point(cam, [0.1, -0.2, 2.0])
    np.testing.assert_allclose(m, [37.0, 14.0])
    assert z == 2.0
    with pytest.raises(errors.PointBehindCamera):
        p.project_point(cam, [0, 0, -1.0])
    # Jacobian vs central differences (reference tests/test_core.py:138-149)
    x = np.array([0.3, -0.1, 3.0])
    j = p.projection_jacobian(cam, x)
    eps = 1e-6
    num = np.stack([(p.project_point(cam, x + eps * e)[0] - p.project_point(cam, x - eps * e)[0])
                    / (2 * eps) for e in np.eye(3)], 1)
    np.testing.assert_allclose(j, num, atol=1e-4)


def test_quaternion_round_trip():
    rng = np.random.default_rng(0)
    for _ in range(200):
        q = p.quat_normalize(rng.normal(size=4))
        q2 = p.matrix_to_quat(p.quat_to_matrix(q))
        assert min(np.linalg.norm(q - q2), np.linalg.norm(q + q2)) < 1e-12


def test_config(tmp_path):
    c = p.Config()
    assert c.alpha_cutoff == 1.0 / 255.0 and c.min_views == 2
    with pytest.raises(errors.InvalidConfig):
        p.Config(alpha_cutoff=0.0)
    with pytest.raises(errors.InvalidConfig):
        p.Config(propagation_average="mode")
    f = tmp_path / "cfg.txt"
    f.write_text("# thresholds\nmin_views = 3\nalpha_cutoff = 0.01\n\n")
    c = p.load_config(f)
    assert c.min_views == 3 and c.alpha_cutoff == 0.01
    f.write_text("bogus = 1\n")
    with pytest.raises(errors.InvalidConfig):
        p.load_config(f)


def test_segment_clips_short_and_long():
    short = p.segment_clips(9, 4, 2, "short")
    assert [c.first_frame for c in short] == [0, 4, 8]
    assert short[0].target_frames == (1, 2, 3) and short[2].target_frames == ()
    long = p.segment_clips(9, 4, 2, "long")
    assert [(c.first_frame, c.target_frames) for c in long] == [(0, (1, 2, 3)), (3, (4, 5, 6)),
                                                                 (6, (7, 8))]
    with pytest.raises(errors.InvalidConfig):
        p.segment_clips(9, 1, 2)


def test_trackfield_validation():
    tf = p.TrackField.identity(0, 4, 3)
    assert tf.target.shape == (3, 4, 2) and tf.valid.all()
    with pytest.raises(ValueError):
        p.TrackField(0, 4, 3, np.zeros((3, 5, 2)), np.ones((3, 4), bool))
    bad = np.zeros((3, 4, 2))
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        p.TrackField(0, 4, 3, bad, np.ones((3, 4), bool))
    valid = np.ones((3, 4), bool)
    valid[0, 0] = False
    p.TrackField(0, 4, 3, bad, valid)  # NaN allowed where invalid


def test_scalar_accumulate_and_lazy_lists():
    acc = MotionAccumulator()
    accumulate(acc, [1.0, 2.0], [1.5, 2.0], 0.5)
    assert acc.pixel_count == 1 and acc.static_pixel_count == 1
    accumulate(acc, [1.0, 2.0], [3.5, 2.0], 0.5)
    assert acc.static_pixel_count == 1
    np.testing.assert_allclose(acc.v1[2, 2], 1.0)
    vml = ViewMotionList(3, [1, 0], np.tile(np.eye(2), (2, 1, 1)), np.zeros((2, 2)),
                         [1.0, 0.0], [5, 0])
    assert len(vml) == 2 and vml[0].status == p.Status.SOLVED
    assert vml[1].status == p.Status.UNSOLVABLE and vml[1].view_id == 3
    ul = MotionUpdateList(np.ones((2, 3)), np.tile([1.0, 0, 0, 0], (2, 1)), np.ones((2, 3)),
                          [1, 0])
    assert [u.status for u in ul] == [p.Status.SOLVED, p.Status.UNSOLVABLE]


def test_gaussian_rows_round_trip():
    gs = [p.Gaussian3D(np.arange(3) + i, [1, i, 0, 0], [0.1, 0.2, 0.3], 0.9) for i in range(4)]
    rows = gaussians_array(gs)
    back = gaussians_from_array(rows)
    for a, b in zip(gs, back):
        np.testing.assert_array_equal(a.mean, b.mean)
        np.testing.assert_allclose(a.rotation, b.rotation, rtol=1e-15)
    gl = GaussianList(rows)
    assert len(gl) == 4 and isinstance(gl[2], p.Gaussian3D)
    new = apply_update_rows(rows, np.ones((4, 3)), rows[:, 3:7], 2 * rows[:, 7:10],
                            np.array([1, 0, 1, 0]))
    np.testing.assert_array_equal(new[1], rows[1])
    np.testing.assert_array_equal(new[0, 0:3], rows[0, 0:3] + 1)


def test_scene_generator_matches_reference():
    d = gd.load("scenes")
    for name, args, kw in [("s7", (7, 2000, 8, 3), dict(mover_fraction=0.3)),
                           ("cfg1", (1, 10_000, 4, 2), dict(focal=180, width=128, height=128,
                                                            scale_range=(0.01, 0.02)))]:
        sc = generate_scene(*args, **kw)
        np.testing.assert_array_equal(cameras_array(sc.cameras), d[name + "_cameras"])
        for t in range(len(sc.frames)):
            np.testing.assert_array_equal(sc.frames[t], d[f"{name}_frame{t}"])


def test_scene_generator_rejects_bad_configs():
    with pytest.raises(errors.InvalidConfig):
        generate_scene(0, 100, 2, 2)
    with pytest.raises(errors.InvalidConfig):
        generate_scene(0, 100, 4, 2, focal=5000)


def test_evaluate_perfect_results_zero_error():
    """evaluate (pipeline.py:273-298) is host-side reporting: exact results have zero error
    (reference tests/test_pipeline.py:142-154)."""
    from paper_2604_02586_b200.pipeline import FrameResult, GaussianList, evaluate
    from paper_2604_02586_b200.scene import generate_scene
    s = generate_scene(13, 80, 4, 4, mover_fraction=0.25, translate_mag=0.02)
    results = [FrameResult(t, GaussianList(s.frames[t]), {"solved": 0, "static": 0,
                                                          "unsolvable": 0},
                           {"tracking": 0, "compensation": 0, "refinement": 0})
               for t in range(s.n_frames)]
    report = evaluate(results, s)
    assert len(report.rows) == s.n_frames
    for row in report.rows:
        assert row["mean_pos_err"] == pytest.approx(0.0, abs=1e-12)
        assert row["mean_rot_err_deg"] == pytest.approx(0.0, abs=1e-5)
        assert row["mean_rel_scale_err"] == pytest.approx(0.0, abs=1e-12)
