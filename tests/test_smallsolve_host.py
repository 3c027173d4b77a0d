"""K4's small solvers (csrc/smallsolve.cuh) compiled for the HOST (tests/native, test-only build)
against the reference fixtures: the same source the GPU runs, checked without a GPU."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_2604_02586_b200 import _native as nat
from paper_2604_02586_b200.core import camera_from_row
from paper_2604_02586_b200.multiview import _vech_block
from tests import golden_data as gd

HERE = os.path.dirname(os.path.abspath(__file__))
P = ctypes.c_void_p


@pytest.fixture(scope="module")
def lib():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "native")], check=True)
    return ctypes.CDLL(os.path.join(HERE, "native", "libsolver_host.so"))


def _ptr(a):
    return P(a.ctypes.data)


def test_triangulate(lib):
    d = gd.load("fuse_kats")
    cams = [camera_from_row(r) for r in d["tri_cams"]]
    for i in range(int(d["n_tri"])):
        rows = []
        for v, o in zip(d[f"t{i}_sel"], d[f"t{i}_obs"]):
            p = cams[v].projection_matrix()
            rows += [o[0] * p[2] - p[0], o[1] * p[2] - p[1]]
        rows = np.ascontiguousarray(rows)
        x = np.zeros(3)
        st = lib.host_triangulate(_ptr(rows), len(rows), _ptr(x))
        assert st == int(d[f"t{i}_st"]), i
        if st:
            np.testing.assert_allclose(x, d[f"t{i}_x"], rtol=1e-7, atol=1e-9)


def test_covariance(lib):
    d = gd.load("fuse_kats")
    for i in range(int(d["n_cov"])):
        lin = np.ascontiguousarray(np.concatenate([_vech_block(m) for m in d[f"c{i}_m"]]))
        rhs = np.ascontiguousarray(np.concatenate(
            [[c[0, 0], 0.5 * (c[0, 1] + c[1, 0]), c[1, 1]] for c in d[f"c{i}_c2"]]))
        x = np.zeros(6)
        st = lib.host_cov3d(_ptr(lin), _ptr(rhs), len(rhs), _ptr(x))
        assert st == int(d[f"c{i}_st"]), i
        if st:
            np.testing.assert_allclose(x, d[f"c{i}_x"], rtol=1e-6, atol=1e-12)


def test_decompose(lib):
    d = gd.load("fuse_kats")
    for i in range(int(d["n_dec"])):
        sig = np.ascontiguousarray(d[f"d{i}_sigma"])
        ref = np.ascontiguousarray(d[f"d{i}_ref"])
        q, s = np.zeros(4), np.zeros(3)
        st = lib.host_decompose(_ptr(sig), _ptr(ref), ctypes.c_double(1e-12), _ptr(q), _ptr(s))
        assert st == int(d[f"d{i}_st"]), i
        if st:
            np.testing.assert_allclose(s, d[f"d{i}_s"], rtol=1e-9)
            assert min(np.linalg.norm(q - d[f"d{i}_q"]), np.linalg.norm(q + d[f"d{i}_q"])) < 1e-7


@pytest.mark.parametrize("scene", ["scene21", "scene7", "cfg1"])
def test_update_all_host(lib, scene):
    d = gd.load(scene)
    g = np.ascontiguousarray(d["gaussians"])
    n, nv = len(g), len(d["cameras"])
    st = np.ascontiguousarray(d["m_status"].astype(np.int8))
    a, b = np.ascontiguousarray(d["m_a"]), np.ascontiguousarray(d["m_b"])
    w = np.ascontiguousarray(d["m_w"])
    c = np.ascontiguousarray(d["m_cnt"].astype(np.int32))
    dl, q, s = np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3))
    ust = np.zeros(n, np.int8)
    cfg = nat.make_config()
    lib.host_update_all(_ptr(g), ctypes.c_int64(n), nat.make_cameras(d["cameras"]), nv,
                        _ptr(st), _ptr(a), _ptr(b), _ptr(w), _ptr(c), ctypes.byref(cfg),
                        _ptr(dl), _ptr(q), _ptr(s), _ptr(ust))
    np.testing.assert_array_equal(ust, d["u_status"])
    ok = ust == 1
    np.testing.assert_allclose(dl[ok], d["u_delta"][ok], rtol=0, atol=1e-12)
    ang = 2 * np.arccos(np.clip(np.abs((q * d["u_rot"]).sum(1)), 0, 1))
    assert ang[ok].max() < 1e-6
    np.testing.assert_allclose(s[ok], d["u_scale"][ok], rtol=1e-10)


@pytest.mark.parametrize("thr", [1.0, 0.5, 2.75, 1e-3, 0.0, -1.0, float("inf"), float("nan")])
def test_static_without_sqrt(lib, thr):
    """sqrt_rn(d0^2 + d1^2) < thr  <=>  d0^2 + d1^2 <= L(thr) (csrc/common.cuh): exact for every
    input, including points on and one ulp around the threshold circle and non-finite tracks."""
    lib.host_static_sq_limit.restype = ctypes.c_double
    lib.host_static_sq_limit.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(7)
    m = 200_000
    px = rng.integers(0, 2000, m).astype(np.int32)
    py = rng.integers(0, 2000, m).astype(np.int32)
    t = thr if np.isfinite(thr) and thr > 0 else 1.0
    ang = rng.uniform(0, 2 * np.pi, m)
    rad = t * (1 + rng.choice([-1, 0, 1], m) * np.ldexp(1.0, -52) * rng.integers(0, 4, m))
    rad[: m // 4] = rng.uniform(0, 3 * t, m // 4)
    u = px + rad * np.cos(ang)
    v = py + rad * np.sin(ang)
    u[:50], v[50:100] = np.nan, np.inf
    a = np.zeros(m, np.uint8)
    b = np.zeros(m, np.uint8)
    lib.host_static_both(_ptr(u), _ptr(v), _ptr(px), _ptr(py), ctypes.c_int64(m),
                         ctypes.c_double(thr), _ptr(a), _ptr(b))
    np.testing.assert_array_equal(a, b)
    if np.isfinite(thr) and thr > 0:
        assert 0 < a.sum() < m
