"""Pin the CPU oracle (oracle/) against the reference-generated golden fixtures.

CPU only.  These tests establish that the checker used by the GPU parity tests reproduces the
reference package's own outputs: bit-exact for the contribution set/order, degenerate ids and
integer counts; rel 1e-12 (alpha) / 1e-9 (T, moments) for libm-vs-numpy exp/log1p.
"""

import numpy as np
import pytest

import oracle
from tests import golden_data as gd

RASTER_KATS = ["peak", "density", "composite", "order", "tie", "earlystop", "degenerate",
               "behind", "edges", "c10_0", "c10_1", "c10_2", "c10_3"]


def _cmp_wm(got, ref):
    for k in ("pixel_x", "pixel_y", "gaussian_id"):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
    np.testing.assert_allclose(got["alpha"], ref["alpha"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(got["transmittance"], ref["transmittance"], rtol=1e-9, atol=0)
    np.testing.assert_array_equal(got["degenerate_ids"], ref["degenerate_ids"])


@pytest.mark.parametrize("name", RASTER_KATS)
def test_raster_kats(name):
    d = gd.load("raster_kats")
    cam = d.get(name + "_camera", d["camera"])
    got = oracle.rasterize(d[name + "_gaussians"], cam)
    _cmp_wm(got, gd.weightmap(d, name + "_"))


def test_raster_cutoff():
    d = gd.load("raster_kats")
    got = oracle.rasterize(d["cutoff_gaussians"], d["camera"], alpha_cutoff=0.5)
    _cmp_wm(got, gd.weightmap(d, "cutoff_"))
    assert np.all(got["alpha"] >= 0.5)


@pytest.mark.parametrize("scene", ["scene21", "scene7", "cfg1"])
def test_scene_raster_accumulate_solve(scene):
    d = gd.load(scene)
    target, valid = gd.tracks(d)
    g = d["gaussians"]
    n = len(g)
    for v, cam in enumerate(d["cameras"]):
        wm = oracle.rasterize(g, cam)
        ref_wm = gd.weightmap(d, f"wm{v}_")
        _cmp_wm(wm, ref_wm)
        acc = oracle.accumulate(wm, target[v], valid[v], n)
        np.testing.assert_array_equal(acc["pixel_count"], d["acc_cnt"][v])
        np.testing.assert_array_equal(acc["static_pixel_count"], d["acc_scnt"][v])
        scale = np.abs(d["acc_v1"][v]).max(axis=(1, 2), keepdims=True) + 1e-300
        np.testing.assert_allclose(acc["v1"] / scale, d["acc_v1"][v] / scale, rtol=0, atol=1e-9)
        np.testing.assert_allclose(acc["v2"] / scale, d["acc_v2"][v] / scale, rtol=0, atol=1e-9)
        np.testing.assert_allclose(acc["weight_sum"], d["acc_w"][v], rtol=1e-9, atol=1e-300)
        # solve on the REFERENCE accumulators must be bit-identical (same LAPACK calls)
        ref_acc = dict(v1=d["acc_v1"][v], v2=d["acc_v2"][v], weight_sum=d["acc_w"][v],
                       pixel_count=d["acc_cnt"][v].astype(np.int64))
        sv = oracle.solve_view(ref_acc)
        np.testing.assert_array_equal(sv["status"], d["m_status"][v])
        np.testing.assert_array_equal(sv["a"], d["m_a"][v])
        np.testing.assert_array_equal(sv["b"], d["m_b"][v])


@pytest.mark.parametrize("scene", ["scene21", "scene7", "cfg1"])
def test_scene_update_all(scene):
    d = gd.load(scene)
    upd = oracle.update_all(d["gaussians"], gd.motions(d), d["cameras"])
    np.testing.assert_array_equal(upd["status"], d["u_status"])
    np.testing.assert_allclose(upd["delta_mean"], d["u_delta"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(upd["rotation"], d["u_rot"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(upd["scale"], d["u_scale"], rtol=1e-12, atol=0)


def test_accumulate_kats():
    d = gd.load("accumulate_kats")
    for i in range(int(d["n_cases"])):
        c = {k[len(f"c{i}_"):]: v for k, v in d.items() if k.startswith(f"c{i}_")}
        wm = dict(pixel_x=c["px"], pixel_y=c["py"], gaussian_id=c["gid"], alpha=c["alpha"],
                  transmittance=c["trans"])
        acc = oracle.accumulate(wm, c["target"], c["valid"], int(c["ng"]))
        np.testing.assert_array_equal(acc["v1"], c["v1"])
        np.testing.assert_array_equal(acc["v2"], c["v2"])
        np.testing.assert_array_equal(acc["weight_sum"], c["w"])
        np.testing.assert_array_equal(acc["pixel_count"], c["cnt"])
        np.testing.assert_array_equal(acc["static_pixel_count"], c["scnt"])
        np.testing.assert_array_equal(acc["static_weight_sum"], c["sw"])
        sv = oracle.solve_view(acc)
        np.testing.assert_array_equal(sv["status"], c["status"])
        np.testing.assert_array_equal(sv["a"], c["a"])
        np.testing.assert_array_equal(sv["b"], c["b"])


def test_binning_restatement_consistent_with_raster():
    """Every kept contribution lies in a binned Gaussian's bbox and tile; tile lists are ordered by
    (depth, gid) exactly as splat.py:178 orders a pixel's contributions."""
    d = gd.load("cfg1")
    g = d["gaussians"]
    for cam in d["cameras"]:
        b = oracle.bin_view(g, cam)
        wm = oracle.rasterize(g, cam)
        _, depth, _, _ = oracle.project(g, cam)
        gid = wm["gaussian_id"]
        assert np.all(b["status"][gid] == 3)
        bb = b["bbox"][gid]
        assert np.all((wm["pixel_x"] >= bb[:, 0]) & (wm["pixel_x"] <= bb[:, 1]))
        assert np.all((wm["pixel_y"] >= bb[:, 2]) & (wm["pixel_y"] <= bb[:, 3]))
        tiles_x = (int(cam[16]) + 15) // 16
        for t in np.flatnonzero(b["tile_count"]):
            s, c = b["tile_start"][t], b["tile_count"][t]
            assert np.all(b["inst_tile"][s:s + c] == t)
            ids = b["inst_gid"][s:s + c]
            key = np.lexsort((ids, depth[ids]))
            assert np.array_equal(key, np.arange(c))
            tx, ty = t % tiles_x, t // tiles_x
            bbt = b["bbox"][ids] // 16
            assert np.all((bbt[:, 0] <= tx) & (tx <= bbt[:, 1]) & (bbt[:, 2] <= ty)
                          & (ty <= bbt[:, 3]))


@pytest.mark.parametrize("scene", ["scene21", "scene7", "cfg1"])
def test_product_transmittance_mode(scene):
    """oracle.rasterize(transmittance="product") (the GPU's exact running product, used by the
    at-scale parity tests) keeps the reference's contribution set on the fixtures, with T within
    the reference's own log-cumsum rounding."""
    d = gd.load(scene)
    for v, cam in enumerate(d["cameras"]):
        got = oracle.rasterize(d["gaussians"], cam, transmittance="product")
        _cmp_wm(got, gd.weightmap(d, f"wm{v}_"))
