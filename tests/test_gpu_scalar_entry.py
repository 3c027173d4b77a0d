"""The scalar and per-view entry points that run on the GPU, against the reference's outputs.

* solve_motion (motion2d.py:99-110; K3 with batch 1): the 200 scalar KATs of
  make_golden.accumulate_kats (reference MotionAccumulator + solve_motion, C2-style);
* update_gaussian (multiview.py:278-315; K4 with N = 1): every Gaussian of the scene21 fixture on
  the reference's own motions vs the reference's update_all (the reference pins batched == scalar
  in tests/test_multiview.py:194-231);
* solve_all_views (motion2d.py:187-204): the reference's scene21 / scene7 weight maps and tracks
  through the GPU accumulate + solve vs the reference's accumulators and motions.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from tests import golden_data as gd  # noqa: E402


def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_solve_motion_scalar_kats():
    _need_cuda()
    from paper_2604_02586_b200.motion2d import MotionAccumulator, Status, solve_motion
    d = gd.load("accumulate_kats")
    n_solved = 0
    for i in range(int(d["n_scalar"])):
        wsum = 0.0
        for w in d[f"s{i}_ws"]:  # the reference's running sum (motion2d.py:90)
            wsum += float(w)
        acc = MotionAccumulator(v1=d[f"s{i}_v1"].copy(), v2=d[f"s{i}_v2"].copy(),
                                weight_sum=wsum, pixel_count=len(d[f"s{i}_ws"]))
        vm = solve_motion(acc, gaussian_id=i, view_id=0)
        st = int(d[f"s{i}_st"])
        assert (vm.status == Status.SOLVED) == bool(st), f"case {i}"
        if st:
            n_solved += 1
            np.testing.assert_allclose(vm.motion.a, d[f"s{i}_ma"], rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(vm.motion.b, d[f"s{i}_mb"], rtol=1e-9, atol=1e-7)
        else:
            np.testing.assert_array_equal(vm.motion.a, np.eye(2))
            np.testing.assert_array_equal(vm.motion.b, np.zeros(2))
    assert n_solved > 100


def _reference_motions(d, v):
    from paper_2604_02586_b200.core import AffineMotion
    from paper_2604_02586_b200.motion2d import Status, ViewMotion
    out = []
    for i in range(len(d["gaussians"])):
        solved = bool(d["m_status"][v, i])
        mot = AffineMotion(d["m_a"][v, i], d["m_b"][v, i]) if solved else AffineMotion.identity()
        out.append(ViewMotion(i, v, mot, float(d["m_w"][v, i]), int(d["m_cnt"][v, i]),
                              Status.SOLVED if solved else Status.UNSOLVABLE))
    return out


def test_update_gaussian_vs_reference_update_all():
    _need_cuda()
    from paper_2604_02586_b200.core import camera_from_row, gaussians_from_array
    from paper_2604_02586_b200.motion2d import Status
    from paper_2604_02586_b200.multiview import update_gaussian
    d = gd.load("scene21")
    gs = gaussians_from_array(d["gaussians"])
    cams = [camera_from_row(r) for r in d["cameras"]]
    per_view = [_reference_motions(d, v) for v in range(len(cams))]
    n_solved = 0
    for i, g in enumerate(gs):
        u = update_gaussian(g, [per_view[v][i] for v in range(len(cams))], cams, gaussian_id=i)
        assert u.gaussian_id == i
        assert (u.status == Status.SOLVED) == bool(d["u_status"][i]), f"Gaussian {i}"
        if u.status == Status.SOLVED:
            n_solved += 1
            np.testing.assert_allclose(u.delta_mean, d["u_delta"][i], atol=1e-9)
            dot = abs(float(np.dot(u.new_rotation, d["u_rot"][i])))
            assert 2 * np.arccos(min(dot, 1.0)) < 1e-7
            np.testing.assert_allclose(u.new_scale, d["u_scale"][i], rtol=1e-9)
        else:
            np.testing.assert_array_equal(u.delta_mean, np.zeros(3))
            np.testing.assert_array_equal(u.new_rotation, g.rotation)
            np.testing.assert_array_equal(u.new_scale, g.scale)
    assert n_solved > 0


@pytest.mark.parametrize("scene", ["scene21", "scene7"])
def test_solve_all_views_vs_reference(scene):
    _need_cuda()
    from paper_2604_02586_b200.errors import DimensionMismatch
    from paper_2604_02586_b200.motion2d import Status, TrackField, solve_all_views
    from paper_2604_02586_b200.splat import WeightMap
    d = gd.load(scene)
    target, valid = gd.tracks(d)
    nv, h, w = valid.shape
    n = len(d["gaussians"])
    wms = []
    for v in range(nv):
        a = gd.weightmap(d, f"wm{v}_")
        wms.append(WeightMap(v, w, h, a["pixel_x"], a["pixel_y"], a["gaussian_id"], a["alpha"],
                             a["transmittance"], np.ones(len(a["alpha"])), a["degenerate_ids"]))
    tfs = [TrackField(v, w, h, target[v], valid[v]) for v in range(nv)]
    motions, accs = solve_all_views(wms, tfs, n)
    assert len(motions) == nv and len(accs) == nv
    for v in range(nv):
        np.testing.assert_array_equal(accs[v].pixel_count, d["acc_cnt"][v])
        np.testing.assert_array_equal(accs[v].static_pixel_count, d["acc_scnt"][v])
        np.testing.assert_allclose(accs[v].weight_sum, d["acc_w"][v], rtol=1e-12, atol=1e-300)
        scale = np.abs(d["acc_v1"][v]).max(axis=(1, 2), keepdims=True) + 1e-300
        np.testing.assert_allclose(accs[v].v1 / scale, d["acc_v1"][v] / scale, atol=1e-12)
        st = np.array([vm.status == Status.SOLVED for vm in motions[v]])
        np.testing.assert_array_equal(st, d["m_status"][v].astype(bool))
        a = np.array([vm.motion.a for vm in motions[v]])
        np.testing.assert_allclose(a[st], d["m_a"][v][st], atol=1e-6)
    with pytest.raises(DimensionMismatch):
        solve_all_views(wms[:1], tfs, n)
