"""patch.install() rebinds the reference pipeline's stage names (CPU: mechanics and type
conversion only; skipped where the reference package is not importable)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def gausstrack():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF)
    try:
        import gausstrack
        return gausstrack
    finally:
        sys.path.remove(REF)


def test_install_rebinds_pipeline_names(gausstrack):
    import gausstrack.pipeline as gp
    import gausstrack.scene as gs

    from paper_2604_02586_b200 import patch
    before = {n: getattr(gp, n) for n in patch._STAGES}
    h = patch.install()
    try:
        for n in patch._STAGES:
            assert getattr(gp, n) is not before[n]
            assert getattr(gp, n).__module__ == "paper_2604_02586_b200.patch"
        assert gs.rasterize_weights.__module__ == "paper_2604_02586_b200.patch"
    finally:
        patch.uninstall(h)
    for n in patch._STAGES:
        assert getattr(gp, n) is before[n]


def test_reference_typed_motions(gausstrack):
    import gausstrack.core as gcore
    import gausstrack.motion2d as gm

    from paper_2604_02586_b200.motion2d import ViewMotionList, motions_arrays
    from paper_2604_02586_b200.patch import to_reference_motions
    vml = ViewMotionList(2, [1, 0, 1], np.tile(np.eye(2), (3, 1, 1)) * 1.5,
                         np.arange(6.0).reshape(3, 2), [1.0, 0.0, 2.0], [4, 0, 9])
    ref = to_reference_motions(vml, gm, gcore)
    assert [vm.status for vm in ref] == [gm.Status.SOLVED, gm.Status.UNSOLVABLE,
                                         gm.Status.SOLVED]
    assert isinstance(ref[0].motion, gcore.AffineMotion) and ref[1].view_id == 2
    # our array extraction accepts the reference's enum (matched by value)
    st, a, b, w, c = motions_arrays(ref)
    np.testing.assert_array_equal(st, [1, 0, 1])
    np.testing.assert_array_equal(b[2], [4.0, 5.0])


def test_reference_typed_inputs_convert(gausstrack):
    """The shims receive the reference's own CameraView / Gaussian3D objects from
    gausstrack.pipeline.compensate_frame: the host layout must accept them field by field."""
    from gausstrack.core import CameraView, Gaussian3D

    from paper_2604_02586_b200.core import cameras_array, gaussians_array
    from tests import golden_data as gd
    d = gd.load("scene21")
    cams = [CameraView(c[:9].reshape(3, 3), c[9:12], c[12], c[13], c[14], c[15], int(c[16]),
                       int(c[17])) for c in d["cameras"]]
    np.testing.assert_array_equal(cameras_array(cams), d["cameras"])
    gs = [Gaussian3D(r[0:3], r[3:7], r[7:10], r[10]) for r in d["gaussians"]]
    want = np.array([np.concatenate([g.mean, g.rotation, g.scale, [g.opacity]]) for g in gs])
    np.testing.assert_array_equal(gaussians_array(gs), want)
