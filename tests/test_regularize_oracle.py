"""Regularisation (regularize.py:37-188) on the CPU:

* the oracle (oracle/regularize.py, oracle.c orc_knn) against the reference's own outputs
  (tests/golden/regularize_kats.npz, made by tests/golden/make_golden.py): kNN bit-exact
  (including distance ties on a lattice with duplicate points), static flags exact, median filter /
  propagation / apply_updates bit-exact or to LAPACK-rounding level;
* the device rotation helpers (csrc/rotation.cuh, compiled for the host in tests/native) against
  scipy's Rotation and numpy/LAPACK: from_matrix / from_euler / as_matrix and the 3x3 products
  bit-exact, as_euler to 1 ulp-level, the polar factor to 1e-12 (noisy, ill-conditioned inputs).
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

from oracle import regularize as oreg
from tests import golden_data as gd

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ("cloud", "lattice")


@pytest.fixture(scope="module")
def kats():
    return gd.load("regularize_kats")


def _in(d, c, pre="in"):
    return tuple(d[f"{c}_{pre}_{t}"] for t in ("delta", "rot", "scale", "status"))


@pytest.mark.parametrize("case", CASES)
def test_knn_bit_exact(kats, case):
    pos = kats[f"{case}_rows"][:, 0:3]
    for k in (8, 3):
        np.testing.assert_array_equal(oreg.knn(pos, k), kats[f"{case}_k{k}_adj"])


def test_knn_edge_cases():
    with pytest.raises(ValueError):
        oreg.knn(np.zeros((1, 3)))
    assert oreg.knn(np.random.default_rng(0).normal(size=(4, 3)), 8).shape == (4, 3)
    pts = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [2, 0, 0.0]])
    assert list(oreg.knn(pts, 2)[0]) == [1, 2]  # tie at distance 1 -> lower id first


@pytest.mark.parametrize("case", CASES)
def test_regularize_matches_reference(kats, case):
    rows = kats[f"{case}_rows"]
    adj = kats[f"{case}_k8_adj"]
    flags = oreg.detect_static_all(kats[f"{case}_pc"], kats[f"{case}_sc"])
    np.testing.assert_array_equal(flags, kats[f"{case}_flags"])
    med = oreg.median_filter(rows, *_in(kats, case), adj)
    for got, ref in zip(med, _in(kats, case, "med")):
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14)
    for avg in ("mean", "median"):
        ref = _in(kats, case, "p" + avg)
        got = oreg.propagate(rows, *_in(kats, case, "med"), adj, flags, avg)
        for g, r in zip(got, ref):
            np.testing.assert_array_equal(g, r)
    out = oreg.apply_updates(rows, *_in(kats, case, "pmean"))
    np.testing.assert_array_equal(out, kats[f"{case}_applied"])
    # the golden sets exercise every branch
    st = kats[f"{case}_pmean_status"]
    assert (st == 0).any() or case == "lattice"
    assert (st == 1).any() and (st == 2).any()
    assert (kats[f"{case}_in_status"] == 0).sum() > (st == 0).sum()  # some were filled


@pytest.fixture(scope="module")
def host():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "native")], check=True)
    return ctypes.CDLL(os.path.join(HERE, "native", "libsolver_host.so"))


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _call(fn, *args, out_shape):
    out = np.zeros(out_shape)
    fn(*[_p(np.ascontiguousarray(a, np.float64)) for a in args], _p(out))
    return out


def test_rotation_helpers_vs_scipy(host):
    rng = np.random.default_rng(5)
    euler_err = 0.0
    for t in range(3000):
        r = Rotation.random(random_state=t)
        m = r.as_matrix()
        q = _call(host.host_sp_from_matrix, m, out_shape=4)
        np.testing.assert_array_equal(q, Rotation.from_matrix(m).as_quat())
        e = _call(host.host_sp_as_euler_xyz, r.as_quat(), out_shape=3)
        euler_err = max(euler_err, np.abs(e - r.as_euler("XYZ")).max())
        ang = rng.uniform(-np.pi, np.pi, 3)
        mm = _call(host.host_sp_euler_xyz_to_matrix, ang, out_shape=9).reshape(3, 3)
        np.testing.assert_array_equal(mm, Rotation.from_euler("XYZ", ang).as_matrix())
        a, b = rng.normal(size=(3, 3)), rng.normal(size=(3, 3))
        np.testing.assert_array_equal(_call(host.host_matmul3, a, b, out_shape=9).reshape(3, 3),
                                      a @ b)
        np.testing.assert_array_equal(
            _call(host.host_matmul3_bt, a, b, out_shape=9).reshape(3, 3), a @ b.T)
    assert euler_err < 1e-15


def test_nearest_rotation_vs_lapack(host):
    rng = np.random.default_rng(6)
    for t in range(2000):
        m = Rotation.random(random_state=t).as_matrix() + rng.normal(0, 0.2, (3, 3))
        if t % 3 == 0:
            m = -m  # det < 0 branch
        got = _call(host.host_nearest_rotation, m, out_shape=9).reshape(3, 3)
        ref = oreg._nearest_rotation(m.copy())
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
        assert np.linalg.det(got) > 0


@pytest.mark.parametrize("scene", ["scene21", "scene7"])
@pytest.mark.parametrize("avg", ["mean", "median"])
def test_oracle_compensate_frame_matches_reference(scene, avg):
    """Oracle hot path + oracle regularisation == the reference's full compensate_frame."""
    import oracle
    d = gd.load(scene)
    ref = gd.load("compensate_kats")
    target, valid = gd.tracks(d)
    g, cams = d["gaussians"], d["cameras"]
    upd, mots, accs = oracle.compensate(g, cams, list(target), list(valid))
    adj = oreg.knn(g[:, 0:3], 8)
    np.testing.assert_array_equal(adj, ref[f"{scene}_knn"])
    pc = np.stack([a["pixel_count"] for a in accs], axis=1)
    sc = np.stack([a["static_pixel_count"] for a in accs], axis=1)
    out = oreg.regularize(g, upd["delta_mean"], upd["rotation"], upd["scale"],
                          upd["status"].astype(np.int8), pc, sc, adj, average=avg)
    st = out[3]
    tallies = [int((st == 1).sum()), int((st == 2).sum()), int((st == 0).sum())]
    np.testing.assert_array_equal(tallies, ref[f"{scene}_{avg}_tallies"])
    # the hot-path stages carry libm-vs-numpy ulp differences in alpha / T (oracle/__init__.py
    # header), which reach the updated parameters at the 1e-9 level
    np.testing.assert_allclose(out[5], ref[f"{scene}_{avg}_rows"], rtol=1e-7, atol=5e-9)
