"""Edge cases of the fused path (K1-K4) against the CPU oracle and the reference's error rules:
all-invalid and NaN-at-invalid tracks, identity tracks, a single Gaussian / single view, images
whose sides are not multiples of the 16-pixel tile, Gaussians behind or outside every camera,
view-count limits and shape errors."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from tests import golden_data as gd  # noqa: E402


@pytest.fixture(scope="module")
def scene7():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    return d["gaussians"], d["cameras"], target, valid


def _run(g, cams, target, valid):
    from paper_2604_02586_b200.engine import FrameEngine
    eng = FrameEngine().bin(g, cams)
    out = eng.compensate(target, valid.astype(np.uint8))
    torch.cuda.synchronize()
    return out


def test_all_invalid_tracks(scene7):
    g, cams, target, valid = scene7
    out = _run(g, cams, target.astype(np.float32), np.zeros_like(valid))
    assert int(out.pixel_count.sum()) == 0 and int(out.static_pixel_count.sum()) == 0
    assert bool((out.motion_status == 0).all()) and bool((out.status == 0).all())
    np.testing.assert_array_equal(out.rotation.cpu().numpy(), g[:, 3:7])
    np.testing.assert_array_equal(out.scale.cpu().numpy(), g[:, 7:10])
    assert float(out.weight_sum.abs().sum()) == 0.0


def test_nan_targets_at_invalid_pixels_are_ignored(scene7):
    """TrackField allows non-finite targets where invalid (motion2d.py:50-51)."""
    g, cams, target, valid = scene7
    t_nan = target.copy()
    t_nan[~valid] = np.nan
    a = _run(g, cams, target, valid)
    b = _run(g, cams, t_nan, valid)
    for k in ("status", "delta_mean", "rotation", "scale", "pixel_count", "weight_sum"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k


def test_identity_tracks_recover_no_motion(scene7):
    g, cams, target, valid = scene7
    v, h, w = valid.shape
    ys, xs = np.mgrid[0:h, 0:w]
    ident = np.broadcast_to(np.stack([xs, ys], -1).astype(np.float32), (v, h, w, 2)).copy()
    out = _run(g, cams, ident, valid)
    st = out.status.cpu().numpy()
    assert (st == 1).sum() > 0.5 * len(g)
    d = out.delta_mean.cpu().numpy()[st == 1]
    assert np.abs(d).max() < 1e-6
    # every tracked pixel is static (|x' - x| = 0 < 1 px)
    np.testing.assert_array_equal(out.static_pixel_count.cpu().numpy(),
                                  out.pixel_count.cpu().numpy())


def test_single_gaussian_and_single_view(scene7):
    g, cams, target, valid = scene7
    out = _run(g[:1], cams[:1], target[:1], valid[:1])
    assert out.status.shape == (1,) and int(out.status[0]) == 0  # min_views = 2
    acc = oracle.accumulate(oracle.rasterize(g[:1], cams[0]), target[0], valid[0], 1)
    assert int(out.pixel_count[0]) == int(acc["pixel_count"][0])


def test_odd_image_size_vs_oracle():
    """37x29 images: partial tiles on the right and bottom edges."""
    from paper_2604_02586_b200.scene import generate_scene, oracle_tracks
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sc = generate_scene(5, 300, 4, 2, focal=30, width=37, height=29, scale_range=(0.02, 0.05))
    tgt, val = oracle_tracks(sc, 1)
    cams = np.array([c.as_row() for c in sc.cameras])
    t_np, v_np = tgt.cpu().numpy().astype(np.float64), val.cpu().numpy().astype(bool)
    out = _run(sc.frames[0], cams, tgt.cpu().numpy(), v_np)
    upd, mots, accs = oracle.compensate(sc.frames[0], cams, list(t_np), list(v_np))
    n = len(sc.frames[0])
    np.testing.assert_array_equal(out.pixel_count.cpu().numpy().reshape(4, n),
                                  np.stack([a["pixel_count"] for a in accs]))
    assert int(out.pixel_count.sum()) > 0
    np.testing.assert_array_equal(out.status.cpu().numpy(), upd["status"])


def test_gaussians_behind_and_outside_cameras(scene7):
    """Gaussians behind every camera or far outside the frustum are never binned and end
    UNSOLVABLE with frame-1 parameters; the rest of the frame is unaffected."""
    g, cams, target, valid = scene7
    extra = g[:3].copy()
    extra[0, 0:3] = [0.0, 0.0, 500.0]    # far above the ring: off every image
    extra[1, 0:3] = [1e4, 1e4, 0.0]      # far away behind / off
    extra[2, 7:10] = 1e-9                # sub-pixel, below the alpha cutoff everywhere
    g2 = np.concatenate([g, extra])
    out = _run(g2, cams, target, valid)
    st = out.status.cpu().numpy()
    assert (st[-3:] == 0).all()
    base = _run(g, cams, target, valid)
    np.testing.assert_array_equal(st[:-3], base.status.cpu().numpy())


def test_argument_errors(scene7):
    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.errors import DimensionMismatch
    g, cams, target, valid = scene7
    eng = FrameEngine().bin(g, cams)
    with pytest.raises(DimensionMismatch):
        eng.compensate(target[:, :-1], valid[:, :-1].astype(np.uint8))
    with pytest.raises(DimensionMismatch):
        eng.compensate(target[:2], valid[:2].astype(np.uint8))
    # more than 64 views: binned as two plans (tests/test_gpu_rigs.py checks the results)
    many = np.repeat(cams[:1], 65, axis=0)
    assert FrameEngine().bin(g[:10], many).grouped


@pytest.mark.parametrize("cap", [1, 2, 3])
def test_k2_residency_cap_is_bit_identical(scene7, cap):
    """ts_plan_set_k2_ctas_per_sm changes only how many warps pull K2's work queue: every
    (tile, quadrant) unit is still walked by one warp in list order, so outputs are bit-identical."""
    from paper_2604_02586_b200.engine import FrameEngine
    g, cams, target, valid = scene7
    a = _run(g, cams, target, valid)
    eng = FrameEngine()
    eng.plan.set_k2_ctas_per_sm(cap)
    eng.bin(g, cams)
    b = eng.compensate(target, valid.astype(np.uint8))
    torch.cuda.synchronize()
    for k in ("status", "delta_mean", "rotation", "scale", "pixel_count", "weight_sum",
              "motion_status", "static_pixel_count"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    with pytest.raises(Exception):
        eng.plan.set_k2_ctas_per_sm(-1)


def test_long_depth_tie_runs_bit_exact():
    """Planar, fronto-parallel geometry: thousands of Gaussians at one exact depth (order by gid,
    splat.py:178) and thousands at depths equal in K1's quantised key but distinct in float64.
    These runs are far longer than the insertion-sort repair handles; they go through the
    segmented sort on exact depth bits.  Binning must equal the oracle bit for bit."""
    import oracle
    from paper_2604_02586_b200.engine import FrameEngine
    rng = np.random.default_rng(3)
    n_flat, n_near, n_rand = 6000, 6000, 8000
    n = n_flat + n_near + n_rand
    g = np.zeros((n, 11))
    g[:, 0] = rng.uniform(-2.0, 2.0, n)
    g[:, 1] = rng.uniform(-1.5, 1.5, n)
    z = np.empty(n)
    z[:n_flat] = 5.0
    z[n_flat:n_flat + n_near] = 5.0 + rng.permutation(n_near) * 1e-13
    z[n_flat + n_near:] = rng.uniform(5.0, 15.0, n_rand)
    g[:, 2] = z
    q = rng.normal(size=(n, 4))
    g[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    g[:, 7:10] = rng.uniform(0.004, 0.01, (n, 3))
    g[:, 10] = 0.9
    cam = np.zeros(18)
    cam[[0, 4, 8]] = 1.0  # R = I, t = 0: depth = z exactly
    cam[12:18] = [500.0, 500.0, 320.0, 240.0, 640, 480]
    eng = FrameEngine().bin(g, cam[None])
    b = eng.binning()
    ref = oracle.bin_view(g, cam)
    np.testing.assert_array_equal(b["status"], ref["status"])
    rng_ = b["tile_range"].astype(np.int64)
    np.testing.assert_array_equal(rng_[:, 1] - rng_[:, 0], ref["tile_count"])
    idx = gd.tile_order_index(rng_)
    np.testing.assert_array_equal(b["inst_gv"][idx].astype(np.int64), ref["inst_gid"])


def test_far_offscreen_gaussians_widen_depth_range_bit_exact():
    """K1's key range comes from every in-front Gaussian (k1_depth_bounds), a superset of the
    binned ones: far-away Gaussians off the image (in front, never binned) stretch the range by
    six orders of magnitude, so most binned depths share quantised keys and the order rests on
    the exact tie repair.  Binning must still equal the oracle bit for bit."""
    import oracle
    from paper_2604_02586_b200.engine import FrameEngine
    rng = np.random.default_rng(5)
    n_vis, n_far = 6000, 50
    n = n_vis + n_far
    g = np.zeros((n, 11))
    g[:n_vis, 0] = rng.uniform(-2.0, 2.0, n_vis)
    g[:n_vis, 1] = rng.uniform(-1.5, 1.5, n_vis)
    g[:n_vis, 2] = rng.uniform(5.0, 5.0 + 1e-6, n_vis)  # a thin slab: ~50 key levels at most
    g[n_vis:, 0] = rng.uniform(1e8, 2e8, n_far)          # far to the side: off the image
    g[n_vis:, 2] = rng.uniform(1e6, 2e6, n_far)
    q = rng.normal(size=(n, 4))
    g[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    g[:, 7:10] = rng.uniform(0.004, 0.01, (n, 3))
    g[:, 10] = 0.9
    cam = np.zeros(18)
    cam[[0, 4, 8]] = 1.0
    cam[12:18] = [500.0, 500.0, 320.0, 240.0, 640, 480]
    eng = FrameEngine().bin(g, cam[None])
    b = eng.binning()
    ref = oracle.bin_view(g, cam)
    np.testing.assert_array_equal(b["status"], ref["status"])
    assert (ref["status"][n_vis:] != 3).all() and (ref["status"][:n_vis] == 3).sum() > 1000
    rng_ = b["tile_range"].astype(np.int64)
    np.testing.assert_array_equal(rng_[:, 1] - rng_[:, 0], ref["tile_count"])
    idx = gd.tile_order_index(rng_)
    np.testing.assert_array_equal(b["inst_gv"][idx].astype(np.int64), ref["inst_gid"])


def test_empty_frame(scene7):
    """No Gaussians (the reference returns empty lists): every stage handles N = 0."""
    from paper_2604_02586_b200.engine import FrameEngine
    _, cams, target, valid = scene7
    eng = FrameEngine().bin(np.zeros((0, 11)), cams)
    out = eng.compensate(target.astype(np.float32), valid.astype(np.uint8))
    torch.cuda.synchronize()
    assert out.status.numel() == 0 and out.motion_status.numel() == 0
    assert out.tallies() == {"solved": 0, "static": 0, "unsolvable": 0}


def test_cache_edge_cases(scene7):
    """The clip contribution cache with no Gaussians, and with every track invalid (every cached
    contribution dropped per frame: all UNSOLVABLE, frame-1 rotation / scale kept)."""
    from paper_2604_02586_b200.engine import FrameEngine
    g, cams, target, valid = scene7
    eng = FrameEngine().bin(np.zeros((0, 11)), cams).build_cache()
    out = eng.compensate(target.astype(np.float32), valid.astype(np.uint8), motions=False)
    torch.cuda.synchronize()
    assert out.status.numel() == 0 and eng.cache_info() == (0, 0)
    eng = FrameEngine().bin(g, cams).build_cache()
    assert eng.cache_info()[1] > 0
    for motions in (True, False):
        out = eng.compensate(target.astype(np.float32), np.zeros_like(valid, dtype=np.uint8),
                             motions=motions)
        torch.cuda.synchronize()
        assert bool((out.status == 0).all())
        np.testing.assert_array_equal(out.rotation.cpu().numpy(), g[:, 3:7])
        if motions:
            assert int(out.pixel_count.sum()) == 0 and bool((out.motion_status == 0).all())
