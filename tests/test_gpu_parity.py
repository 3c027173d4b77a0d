"""GPU parity: the CUDA path (through the C ABI) against the oracle and the reference goldens.

Tolerance contract:
  * projection mean2/depth/cov2, bbox, binning keys / instance order / tile ranges, contribution
    set and order, degenerate ids, pixel and static counts: bit-exact;
  * alpha: rel 1e-12; transmittance (product vs the reference's log-cumsum): rel 1e-9;
  * moments / weight sums: rel 1e-9 of the row scale;
  * per-view status flips: <= 1e-4 of eligible fits (listed); moved mean A mu + b: 1e-6 px;
  * update means: rel 1e-4, rotations 1e-3 rad (scale gap >= 5%), scales rel 1e-4, for
    >= 99.99% of SOLVED Gaussians.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from tests import golden_data as gd  # noqa: E402

SCENES = ["scene21", "scene7", "cfg1"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_02586_b200 import _native
    _native.lib()  # fails loudly if the library is not built


def _project_gpu(g, cam):
    import ctypes

    from paper_2604_02586_b200 import _native as nat
    n = len(g)
    dg = torch.as_tensor(np.ascontiguousarray(g), device="cuda")
    mean2 = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    depth = torch.empty(n, dtype=torch.float64, device="cuda")
    cov2 = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    inf = torch.empty(n, dtype=torch.uint8, device="cuda")
    c = nat.make_camera(cam)
    nat.check(nat.lib().ts_project(nat.dptr(dg), n, ctypes.byref(c), nat.dptr(mean2),
                                   nat.dptr(depth), nat.dptr(cov2), nat.dptr(inf),
                                   nat.stream_ptr()))
    return (mean2.cpu().numpy(), depth.cpu().numpy(), cov2.cpu().numpy(),
            inf.cpu().numpy().astype(bool))


@pytest.mark.parametrize("scene", SCENES)
def test_projection_bit_exact(scene):
    d = gd.load(scene)
    for cam in d["cameras"]:
        got = _project_gpu(d["gaussians"], cam)
        ref = oracle.project(d["gaussians"], cam)
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("scene", SCENES)
def test_binning_bit_exact(scene):
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load(scene)
    g, cams = d["gaussians"], d["cameras"]
    n = len(g)
    eng = FrameEngine().bin(g, cams)
    b = eng.binning()
    tpv = b["tiles_x"] * b["tiles_y"]
    for v, cam in enumerate(cams):
        ref = oracle.bin_view(g, cam)
        np.testing.assert_array_equal(b["status"][v * n:(v + 1) * n], ref["status"])
        st3 = ref["status"] == 3
        np.testing.assert_array_equal(b["bbox"][v * n:(v + 1) * n][st3], ref["bbox"][st3])
        rng = b["tile_range"][v * tpv:(v + 1) * tpv].astype(np.int64)
        cnt = rng[:, 1] - rng[:, 0]
        np.testing.assert_array_equal(cnt, ref["tile_count"])
        idx = gd.tile_order_index(rng)  # the view's instances, tile-major
        np.testing.assert_array_equal(b["inst_tile"][idx].astype(np.int64), ref["inst_tile"])
        np.testing.assert_array_equal(b["inst_gv"][idx].astype(np.int64) - v * n,
                                      ref["inst_gid"])


def _cmp_wm(got, ref):
    np.testing.assert_array_equal(got.pixel_x, ref["pixel_x"])
    np.testing.assert_array_equal(got.pixel_y, ref["pixel_y"])
    np.testing.assert_array_equal(got.gaussian_id, ref["gaussian_id"])
    np.testing.assert_allclose(got.alpha, ref["alpha"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(got.transmittance, ref["transmittance"], rtol=1e-9, atol=0)
    assert list(got.degenerate_ids) == [int(i) for i in ref["degenerate_ids"]]


@pytest.mark.parametrize("name", ["peak", "density", "composite", "order", "tie", "earlystop",
                                  "degenerate", "behind", "edges", "c10_0", "c10_1", "c10_2",
                                  "c10_3"])
def test_rasterize_weights_kats(name):
    from paper_2604_02586_b200.core import camera_from_row
    from paper_2604_02586_b200.splat import rasterize_weights
    d = gd.load("raster_kats")
    cam = camera_from_row(d.get(name + "_camera", d["camera"]))
    wm = rasterize_weights(cam, d[name + "_gaussians"], view_id=3)
    _cmp_wm(wm, gd.weightmap(d, name + "_"))
    assert wm.view_id == 3
    # compositing identity, tests/test_splat.py:56-68
    pix = wm.pixel_y.astype(np.int64) * wm.width + wm.pixel_x
    for p in np.unique(pix):
        msk = pix == p
        lhs = np.sum(wm.alpha[msk] * wm.transmittance[msk])
        assert abs(lhs - (1.0 - np.prod(1.0 - wm.alpha[msk]))) <= 1e-12


def test_rasterize_cutoff_and_errors():
    from paper_2604_02586_b200.core import camera_from_row
    from paper_2604_02586_b200.splat import rasterize_weights
    d = gd.load("raster_kats")
    cam = camera_from_row(d["camera"])
    wm = rasterize_weights(cam, d["cutoff_gaussians"], alpha_cutoff=0.5)
    _cmp_wm(wm, gd.weightmap(d, "cutoff_"))
    with pytest.raises(ValueError):
        rasterize_weights(cam, d["cutoff_gaussians"], alpha_cutoff=0.0)
    assert len(rasterize_weights(cam, [])) == 0


@pytest.mark.parametrize("scene", SCENES)
def test_rasterize_weights_scenes(scene):
    from paper_2604_02586_b200.core import camera_from_row
    from paper_2604_02586_b200.splat import rasterize_weights
    d = gd.load(scene)
    for v, row in enumerate(d["cameras"]):
        wm = rasterize_weights(camera_from_row(row), d["gaussians"], view_id=v)
        _cmp_wm(wm, gd.weightmap(d, f"wm{v}_"))


def test_accumulate_view_bit_exact_kats():
    from paper_2604_02586_b200.motion2d import TrackField, accumulate_view, solve_view
    from paper_2604_02586_b200.splat import WeightMap
    d = gd.load("accumulate_kats")
    for i in range(int(d["n_cases"])):
        c = {k[len(f"c{i}_"):]: v for k, v in d.items() if k.startswith(f"c{i}_")}
        side = c["valid"].shape[0]
        m = len(c["px"])
        wm = WeightMap(0, side, side, c["px"], c["py"], c["gid"], c["alpha"], c["trans"],
                       np.ones(m))
        tf = TrackField(0, side, side, c["target"], c["valid"].astype(bool))
        acc = accumulate_view(wm, tf, int(c["ng"]))
        np.testing.assert_array_equal(acc.v1, c["v1"])
        np.testing.assert_array_equal(acc.v2, c["v2"])
        np.testing.assert_array_equal(acc.weight_sum, c["w"])
        np.testing.assert_array_equal(acc.pixel_count, c["cnt"])
        np.testing.assert_array_equal(acc.static_pixel_count, c["scnt"])
        np.testing.assert_array_equal(acc.static_weight_sum, c["sw"])
        vms = solve_view(acc)
        st = np.array([vm.status.value == "solved" for vm in vms], np.int8)
        np.testing.assert_array_equal(st, c["status"])
        ok = st == 1
        np.testing.assert_allclose(vms.a[ok], c["a"][ok], rtol=1e-8, atol=1e-9)
        np.testing.assert_allclose(vms.b[ok], c["b"][ok], rtol=1e-8, atol=1e-7)


@pytest.mark.parametrize("scene", SCENES)
def test_accumulate_solve_scenes(scene):
    from paper_2604_02586_b200.motion2d import TrackField, accumulate_view, solve_view
    from paper_2604_02586_b200.splat import WeightMap
    d = gd.load(scene)
    target, valid = gd.tracks(d)
    n = len(d["gaussians"])
    h, w = valid.shape[1:]
    for v in range(len(d["cameras"])):
        r = gd.weightmap(d, f"wm{v}_")
        wm = WeightMap(v, w, h, r["pixel_x"], r["pixel_y"], r["gaussian_id"], r["alpha"],
                       r["transmittance"], np.zeros(len(r["alpha"])))
        acc = accumulate_view(wm, TrackField(v, w, h, target[v], valid[v]), n)
        np.testing.assert_array_equal(acc.v1, d["acc_v1"][v])
        np.testing.assert_array_equal(acc.v2, d["acc_v2"][v])
        np.testing.assert_array_equal(acc.pixel_count, d["acc_cnt"][v])
        np.testing.assert_array_equal(acc.static_pixel_count, d["acc_scnt"][v])
        vms = solve_view(acc)
        flips = np.flatnonzero(vms.status != d["m_status"][v])
        assert len(flips) <= max(1, 1e-4 * n), f"view {v} status flips {flips}"
        both = (vms.status == 1) & (d["m_status"][v] == 1)
        # compare the moved means A mu + b at the Gaussians' projections
        mu = oracle.project(d["gaussians"], d["cameras"][v])[0]
        got = np.einsum("nij,nj->ni", vms.a, mu) + vms.b
        ref = np.einsum("nij,nj->ni", d["m_a"][v], mu) + d["m_b"][v]
        np.testing.assert_allclose(got[both], ref[both], rtol=0, atol=1e-6)


def _update_stats(st, delta, rot, scale, ref_st, ref_delta, ref_rot, ref_scale, g):
    both = (st == 1) & (ref_st == 1)
    mean = g[:, 0:3]
    rel_mean = (np.linalg.norm((mean + delta) - (mean + ref_delta), axis=1)
                / np.maximum(np.linalg.norm(mean + ref_delta, axis=1), 1e-12))
    ang = 2 * np.arccos(np.clip(np.abs(np.sum(rot * ref_rot, axis=1)), 0, 1))
    srel = np.max(np.abs(scale - ref_scale) / ref_scale, axis=1)
    s_sorted = np.sort(ref_scale, axis=1)
    gap = np.min(np.diff(s_sorted, axis=1) / s_sorted[:, 1:], axis=1)
    return both, rel_mean, ang, srel, gap


def _check_updates(st, delta, rot, scale, ref_st, ref_delta, ref_rot, ref_scale, g,
                   max_status_flip_frac=1e-4):
    n = len(st)
    flips = np.flatnonzero(st != ref_st)
    assert len(flips) <= max(2, max_status_flip_frac * n), f"update status flips: {flips[:20]}"
    both, rel_mean, ang, srel, gap = _update_stats(st, delta, rot, scale, ref_st, ref_delta,
                                                   ref_rot, ref_scale, g)
    k = int(both.sum())
    bad_mean = np.flatnonzero(both & (rel_mean > 1e-4))
    bad_scale = np.flatnonzero(both & (srel > 1e-4))
    bad_rot = np.flatnonzero(both & (gap >= 0.05) & (ang > 1e-3))
    allowed = max(1, int(1e-4 * k))
    assert len(bad_mean) <= allowed, f"mean outliers {bad_mean[:10]}"
    assert len(bad_scale) <= allowed, f"scale outliers {bad_scale[:10]}"
    assert len(bad_rot) <= allowed, f"rotation outliers {bad_rot[:10]}"
    unsolved = st == 0
    np.testing.assert_array_equal(delta[unsolved], 0.0)
    np.testing.assert_array_equal(rot[unsolved], g[unsolved, 3:7])
    np.testing.assert_array_equal(scale[unsolved], g[unsolved, 7:10])


@pytest.mark.parametrize("scene", SCENES)
def test_update_all_on_reference_motions(scene):
    from paper_2604_02586_b200.multiview import update_arrays
    d = gd.load(scene)
    m = gd.motions(d)
    dl, q, s, st = update_arrays(d["gaussians"], d["cameras"], m["status"], m["a"], m["b"],
                                 m["weight_sum"], m["pixel_count"])
    _check_updates(st, dl, q, s, d["u_status"], d["u_delta"], d["u_rot"], d["u_scale"],
                   d["gaussians"], max_status_flip_frac=1e-4)


@pytest.mark.parametrize("scene", SCENES)
def test_fused_frame_vs_oracle(scene):
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load(scene)
    target, valid = gd.tracks(d)
    g, cams = d["gaussians"], d["cameras"]
    n, nv = len(g), len(cams)
    eng = FrameEngine().bin(g, cams)
    out = eng.compensate(target.astype(np.float32), valid.astype(np.uint8))
    torch.cuda.synchronize()
    upd, mots, accs = oracle.compensate(g, cams, list(target), list(valid))
    # integer outputs of the fused raster-accumulate: bit-exact
    np.testing.assert_array_equal(out.pixel_count.cpu().numpy().reshape(nv, n),
                                  np.stack([a["pixel_count"] for a in accs]))
    np.testing.assert_array_equal(out.static_pixel_count.cpu().numpy().reshape(nv, n),
                                  np.stack([a["static_pixel_count"] for a in accs]))
    ref_w = np.stack([a["weight_sum"] for a in accs])
    np.testing.assert_allclose(out.weight_sum.cpu().numpy().reshape(nv, n), ref_w, rtol=1e-9,
                               atol=1e-300)
    ref_sw = np.stack([a["static_weight_sum"] for a in accs])
    np.testing.assert_allclose(out.static_weight_sum.cpu().numpy().reshape(nv, n), ref_sw,
                               rtol=1e-9, atol=1e-300)
    ms = out.motion_status.cpu().numpy().reshape(nv, n)
    ref_ms = np.stack([m["status"] for m in mots])
    flips = np.argwhere(ms != ref_ms)
    assert len(flips) <= max(1, 1e-4 * n * nv), f"per-view status flips {flips[:10]}"
    _check_updates(out.status.cpu().numpy(), out.delta_mean.cpu().numpy(),
                   out.rotation.cpu().numpy(), out.scale.cpu().numpy(), upd["status"],
                   upd["delta_mean"], upd["rotation"], upd["scale"], g)


def test_fused_deterministic():
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    eng = FrameEngine().bin(d["gaussians"], d["cameras"])
    a = eng.compensate(target.astype(np.float32), valid.astype(np.uint8))
    b = eng.compensate(target.astype(np.float32), valid.astype(np.uint8))
    for k in ("delta_mean", "rotation", "scale", "weight_sum", "motion_a", "motion_b"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k


def test_compensate_frame_api():
    from paper_2604_02586_b200 import Config, compensate_frame
    from paper_2604_02586_b200.core import camera_from_row, gaussians_from_array
    from paper_2604_02586_b200.motion2d import TrackField
    d = gd.load("scene21")
    target, valid = gd.tracks(d)
    frame1 = gaussians_from_array(d["gaussians"])
    cams = [camera_from_row(r) for r in d["cameras"]]
    h, w = valid.shape[1:]
    tracks = [TrackField(v, w, h, target[v], valid[v]) for v in range(len(cams))]
    res = compensate_frame(frame1, cams, tracks, Config(), frame_index=1, regularize=False)
    assert res.frame == 1 and len(res.gaussians) == len(frame1)
    assert sum(res.tallies.values()) == len(frame1)
    assert res.tallies["solved"] == int(d["u_status"].sum())


def test_scalar_fuse_kats():
    from paper_2604_02586_b200.core import camera_from_row
    from paper_2604_02586_b200.errors import GaussTrackError
    from paper_2604_02586_b200.multiview import (decompose_covariance, solve_covariance3d,
                                                 triangulate_mean)
    d = gd.load("fuse_kats")
    cams = [camera_from_row(r) for r in d["tri_cams"]]
    for i in range(int(d["n_tri"])):
        obs = [(cams[v], o) for v, o in zip(d[f"t{i}_sel"], d[f"t{i}_obs"])]
        if int(d[f"t{i}_st"]):
            np.testing.assert_allclose(triangulate_mean(obs), d[f"t{i}_x"], rtol=1e-7, atol=1e-9)
        else:
            with pytest.raises(GaussTrackError):
                triangulate_mean(obs)
    for i in range(int(d["n_cov"])):
        obs = list(zip(d[f"c{i}_m"], d[f"c{i}_c2"]))
        if int(d[f"c{i}_st"]):
            np.testing.assert_allclose(solve_covariance3d(obs).vech(), d[f"c{i}_x"], rtol=1e-6,
                                       atol=1e-12)
        else:
            with pytest.raises(GaussTrackError):
                solve_covariance3d(obs)
    for i in range(int(d["n_dec"])):
        if int(d[f"d{i}_st"]):
            q, s = decompose_covariance(d[f"d{i}_sigma"], d[f"d{i}_ref"], None)
            np.testing.assert_allclose(s, d[f"d{i}_s"], rtol=1e-9)
            assert min(np.linalg.norm(q - d[f"d{i}_q"]), np.linalg.norm(q + d[f"d{i}_q"])) < 1e-7
        else:
            with pytest.raises(GaussTrackError):
                decompose_covariance(d[f"d{i}_sigma"], d[f"d{i}_ref"], None)
