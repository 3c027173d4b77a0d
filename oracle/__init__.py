"""CPU oracle for the gausstrack motion-estimation hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  It is the checker, never the product: the
product path (``paper_2604_02586_b200``) runs on the GPU and fails loudly without its CUDA library.

Parity status: PINNED.  ``tests/golden/make_golden.py`` ran the reference package
(``/root/reference/pkg/src/gausstrack``) in the build container and committed its outputs under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this oracle against them:

* projection (``splat.py:80-110``), bbox / degenerate ids (``splat.py:131-146``), the contribution
  set and order (``splat.py:171-180``) and the integer counts of ``accumulate_view``
  (``motion2d.py:154-160``) are bit-exact;
* alpha / transmittance agree to rel 1e-12 / 1e-9 (libm vs numpy's SIMD ``exp``/``log1p``);
* ``solve_view`` (``motion2d.py:164-184``) and ``update_all`` (``multiview.py:168-275``) are
  restated with the same numpy/LAPACK calls, batched over Gaussians with equal solved-view counts.

Layout conventions (shared with the GPU package):
  gaussians  (N, 11) float64: mean[3], unit quaternion (w, x, y, z)[4], scale[3], opacity
  camera     (18,) float64: R[9] (world->camera, row-major), t[3], fx, fy, cx, cy, width, height
  motions    dict of (V, N, ...) arrays: status (1 = SOLVED, 0 = UNSOLVABLE), a (2, 2), b (2),
             weight_sum, pixel_count
"""

from __future__ import annotations

import ctypes
import itertools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STATUS_UNSOLVABLE = 0
STATUS_SOLVED = 1
STATUS_STATIC = 2

_SINGULAR_GAP_REL = 1e-9  # multiview.py:28


def build():
    """Compile liboracle.so from oracle.c (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        i64, dbl, ptr = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        lib.orc_project.argtypes = [i64, ptr, ptr, ptr, ptr, ptr, ptr]
        lib.orc_project.restype = None
        lib.orc_rasterize.argtypes = [i64, ptr, ptr, dbl, dbl, i64, ptr, ptr, ptr, ptr, ptr, ptr,
                                      ptr, ptr, ctypes.c_int]
        lib.orc_rasterize.restype = i64
        lib.orc_bin.argtypes = [i64, ptr, ptr, ctypes.c_int, i64, ptr, ptr, ptr, ptr, ptr, ptr]
        lib.orc_bin.restype = i64
        lib.orc_accumulate.argtypes = [i64, ptr, ptr, ptr, ptr, ptr, ctypes.c_int, ctypes.c_int,
                                       ptr, ptr, i64, dbl, ptr, ptr, ptr, ptr, ptr, ptr]
        lib.orc_accumulate.restype = None
        lib.orc_fit_hp.argtypes = [i64, ptr, ptr, ptr, ptr, ptr, ctypes.c_int, ptr, ptr, i64, dbl,
                                   i64, dbl, ptr, ptr, ptr, ptr, ptr]
        lib.orc_fit_hp.restype = None
        lib.orc_knn.argtypes = [i64, ptr, ctypes.c_int, ptr]
        lib.orc_knn.restype = None
        lib.orc_knn_queries.argtypes = [i64, ptr, ctypes.c_int, i64, ptr, ptr]
        lib.orc_knn_queries.restype = None
        _LIB = lib
    return _LIB


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# projection / raster / binning / accumulate  (C restatement)

def project(gaussians, camera):
    """splat.py:80-110.  Returns mean2 (N,2), depth (N,), cov2 (N,3: xx,xy,yy), in_front (N,)."""
    g = _c(gaussians, np.float64).reshape(-1, 11)
    cam = _c(camera, np.float64)
    n = len(g)
    mean2 = np.empty((n, 2))
    depth = np.empty(n)
    cov2 = np.empty((n, 3))
    inf = np.empty(n, np.uint8)
    _lib().orc_project(n, _p(g), _p(cam), _p(mean2), _p(depth), _p(cov2), _p(inf))
    return mean2, depth, cov2, inf.astype(bool)


def rasterize(gaussians, camera, alpha_cutoff=1.0 / 255.0, early_stop=1e-4,
              transmittance="reference"):
    """splat.py:113-195.  Returns a dict of WeightMap arrays plus degenerate_ids.
    transmittance="reference": the view-global log1p/cumsum T of splat.py:182-191;
    "product": the exact running product per pixel (the GPU's compositing order)."""
    t_mode = {"reference": 0, "product": 1}[transmittance]
    g = _c(gaussians, np.float64).reshape(-1, 11)
    cam = _c(camera, np.float64)
    n = len(g)
    cap = max(1024, 64 * n)
    deg = np.empty(max(n, 1), np.int64)
    ndeg = ctypes.c_int64(0)
    while True:
        px = np.empty(cap, np.int32)
        py = np.empty(cap, np.int32)
        gid = np.empty(cap, np.int64)
        al = np.empty(cap)
        tr = np.empty(cap)
        de = np.empty(cap)
        m = _lib().orc_rasterize(n, _p(g), _p(cam), alpha_cutoff, early_stop, cap, _p(px),
                                 _p(py), _p(gid), _p(al), _p(tr), _p(de), _p(deg),
                                 ctypes.byref(ndeg), t_mode)
        if m <= cap:
            break
        cap = m
    return dict(pixel_x=px[:m].copy(), pixel_y=py[:m].copy(), gaussian_id=gid[:m].copy(),
                alpha=al[:m].copy(), transmittance=tr[:m].copy(), depth=de[:m].copy(),
                degenerate_ids=deg[:ndeg.value].copy())


def bin_view(gaussians, camera, tile_size=16):
    """Tile binning restatement (bbox rule splat.py:139-146, order splat.py:178).

    Returns status (N,) int8 (0 behind, 1 degenerate, 2 empty bbox, 3 binned), bbox (N,4)
    x0 x1 y0 y1, inst_tile / inst_gid (sorted by tile, depth, gid), tile_start / tile_count.
    """
    g = _c(gaussians, np.float64).reshape(-1, 11)
    cam = _c(camera, np.float64)
    n = len(g)
    w, h = int(cam[16]), int(cam[17])
    ntiles = ((w + tile_size - 1) // tile_size) * ((h + tile_size - 1) // tile_size)
    status = np.empty(n, np.int8)
    bbox = np.empty((n, 4), np.int32)
    ts = np.empty(ntiles, np.int64)
    tc = np.empty(ntiles, np.int64)
    cap = max(1024, 4 * n)
    while True:
        it = np.empty(cap, np.int64)
        ig = np.empty(cap, np.int64)
        m = _lib().orc_bin(n, _p(g), _p(cam), tile_size, cap, _p(status), _p(bbox), _p(it),
                           _p(ig), _p(ts), _p(tc))
        if m <= cap:
            break
        cap = m
    return dict(status=status, bbox=bbox, inst_tile=it[:m].copy(), inst_gid=ig[:m].copy(),
                tile_start=ts, tile_count=tc)


def accumulate(wm, target, valid, n_gaussians, static_threshold_px=1.0):
    """motion2d.py:126-161 over WeightMap arrays `wm` (dict) and a (H,W,2) f64 target."""
    target = _c(target, np.float64)
    valid = _c(valid, np.uint8)
    h, w = valid.shape
    n = int(n_gaussians)
    px = _c(wm["pixel_x"], np.int32)
    py = _c(wm["pixel_y"], np.int32)
    gid = _c(wm["gaussian_id"], np.int64)
    al = _c(wm["alpha"], np.float64)
    tr = _c(wm["transmittance"], np.float64)
    v1 = np.empty((n, 3, 3))
    v2 = np.empty((n, 3, 2))
    ws = np.empty(n)
    cnt = np.empty(n, np.int64)
    scnt = np.empty(n, np.int64)
    sws = np.empty(n)
    _lib().orc_accumulate(len(px), _p(px), _p(py), _p(gid), _p(al), _p(tr), w, h, _p(target),
                          _p(valid), n, static_threshold_px, _p(v1), _p(v2), _p(ws), _p(cnt),
                          _p(scnt), _p(sws))
    return dict(v1=v1, v2=v2, weight_sum=ws, pixel_count=cnt, static_pixel_count=scnt,
                static_weight_sum=sws)


def fit_hp(wm, target, valid, n_gaussians, mu, det_floor=1e-12, min_pixels=3, min_weight=1e-3):
    """accumulate_view + solve_view (motion2d.py:126-184) in long double around an anchor pixel:
    the precision yardstick for at-scale fit comparisons (see orc_fit_hp).  mu: (N, 2) means.
    Returns status (N,) int8, a (N,2,2), b (N,2), moved (N,2) = A mu + b."""
    target = _c(target, np.float64)
    valid = _c(valid, np.uint8)
    w = valid.shape[1]
    n = int(n_gaussians)
    mu = _c(mu, np.float64).reshape(n, 2)
    st = np.empty(n, np.int8)
    a = np.empty((n, 2, 2))
    b = np.empty((n, 2))
    moved = np.empty((n, 2))
    _lib().orc_fit_hp(len(wm["pixel_x"]), _p(_c(wm["pixel_x"], np.int32)),
                      _p(_c(wm["pixel_y"], np.int32)), _p(_c(wm["gaussian_id"], np.int64)),
                      _p(_c(wm["alpha"], np.float64)), _p(_c(wm["transmittance"], np.float64)), w,
                      _p(target), _p(valid), n, det_floor, int(min_pixels), min_weight, _p(mu),
                      _p(st), _p(a), _p(b), _p(moved))
    return dict(status=st, a=a, b=b, moved=moved)


# ---------------------------------------------------------------------------
# solve_view / update_all  (numpy restatement, same LAPACK calls as the reference)

def solve_view(acc, det_floor=1e-12, min_pixels=3, min_weight=1e-3):
    """motion2d.py:164-184, returning arrays instead of ViewMotion objects."""
    v1, v2 = acc["v1"], acc["v2"]
    g = len(acc["weight_sum"])
    det = np.linalg.det(v1) if g else np.empty(0)
    solvable = ((acc["pixel_count"] >= min_pixels) & (acc["weight_sum"] >= min_weight)
                & (det >= det_floor))
    ab = np.zeros((g, 3, 2))
    if np.any(solvable):
        ab[solvable] = np.linalg.solve(v1[solvable], v2[solvable])
    a = np.broadcast_to(np.eye(2), (g, 2, 2)).copy()
    b = np.zeros((g, 2))
    a[solvable] = np.transpose(ab[solvable, :2, :], (0, 2, 1))
    b[solvable] = ab[solvable, 2, :]
    return dict(status=solvable.astype(np.int8), a=a, b=b, weight_sum=acc["weight_sum"].copy(),
                pixel_count=acc["pixel_count"].copy(), det=det)


def _quat_to_matrix_batch(q):
    """core.py:31-38, elementwise over (N,4) (no contraction, same bits as the scalar form)."""
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    r = np.empty((len(q), 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - w * z)
    r[:, 0, 2] = 2 * (x * z + w * y)
    r[:, 1, 0] = 2 * (x * y + w * z)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - w * x)
    r[:, 2, 0] = 2 * (x * z - w * y)
    r[:, 2, 1] = 2 * (y * z + w * x)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def _projection_matrix(cam):
    """core.py:140-148 K @ [R | t]."""
    r = cam[:9].reshape(3, 3)
    t = cam[9:12].reshape(3, 1)
    k = np.array([[cam[12], 0.0, cam[14]], [0.0, cam[13], cam[15]], [0.0, 0.0, 1.0]])
    return k @ np.hstack([r, t])


def _vech_linearization(m):
    """multiview.py:138-156."""
    m0, m1 = m[..., 0, :], m[..., 1, :]
    cols = []
    for i, j in [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]:
        if i == j:
            cols.append(np.stack([m0[..., i] * m0[..., i], m0[..., i] * m1[..., i],
                                  m1[..., i] * m1[..., i]], axis=-1))
        else:
            cols.append(np.stack([2.0 * m0[..., i] * m0[..., j],
                                  m0[..., i] * m1[..., j] + m0[..., j] * m1[..., i],
                                  2.0 * m1[..., i] * m1[..., j]], axis=-1))
    return np.stack(cols, axis=-1)


def _min_eig_ok(cov2):
    """multiview.py:159-165."""
    tr = cov2[..., 0, 0] + cov2[..., 1, 1]
    det = cov2[..., 0, 0] * cov2[..., 1, 1] - cov2[..., 0, 1] * cov2[..., 1, 0]
    min_eig = 0.5 * (tr - np.sqrt(np.maximum(tr * tr - 4 * det, 0.0)))
    return min_eig >= -1e-9 * np.maximum(tr, 0.0)


def _quat_normalize(q):
    return q / np.linalg.norm(q)


def _matrix_to_quat(m):
    """core.py:41-62."""
    t = np.trace(m)
    if t > 0:
        s = np.sqrt(t + 1.0) * 2
        q = np.array([0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s,
                      (m[1, 0] - m[0, 1]) / s])
    else:
        i = int(np.argmax(np.diag(m)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = np.sqrt(max(m[i, i] - m[j, j] - m[k, k] + 1.0, 0.0)) * 2
        q = np.empty(4)
        q[0] = (m[k, j] - m[j, k]) / s
        q[1 + i] = 0.25 * s
        q[1 + j] = (m[j, i] + m[i, j]) / s
        q[1 + k] = (m[k, i] + m[i, k]) / s
    if q[0] < 0:
        q = -q
    return _quat_normalize(q)


_PERMS = list(itertools.permutations(range(3)))


def _decompose(sol, ref_quat, eig_floor):
    """multiview.py:103-135 on one vech solution; returns (quat, scale) or None on failure."""
    m = np.array([[sol[0], sol[1], sol[2]], [sol[1], sol[3], sol[4]], [sol[2], sol[4], sol[5]]])
    m = 0.5 * (m + m.T)
    evals, evecs = np.linalg.eigh(m)
    floor = eig_floor * abs(np.trace(m))
    if np.any(evals < floor):
        return None
    ref = _quat_to_matrix_batch(_quat_normalize(ref_quat)[None])[0]
    dots = np.abs(ref.T @ evecs)
    best = max(_PERMS, key=lambda p: sum(dots[k, p[k]] for k in range(3)))
    r = np.empty((3, 3))
    scale = np.empty(3)
    for k in range(3):
        e = evecs[:, best[k]]
        if np.dot(e, ref[:, k]) < 0:
            e = -e
        r[:, k] = e
        scale[k] = np.sqrt(evals[best[k]])
    if np.linalg.det(r) < 0:
        r[:, 2] = -r[:, 2]
    return _matrix_to_quat(r), scale


def _decompose_batch(sols, ref_quats, eig_floor):
    """_decompose over (G, 6) solutions: eigh / det as stacked gufunc calls, the permutation
    search and quaternion branches vectorised, norms and dots per row (the BLAS calls the scalar
    form makes).  Returns (quat (G,4), scale (G,3), ok (G,) bool); same bits as _decompose."""
    g = len(sols)
    m = np.empty((g, 3, 3))
    m[:, 0, 0], m[:, 0, 1], m[:, 0, 2] = sols[:, 0], sols[:, 1], sols[:, 2]
    m[:, 1, 0], m[:, 1, 1], m[:, 1, 2] = sols[:, 1], sols[:, 3], sols[:, 4]
    m[:, 2, 0], m[:, 2, 1], m[:, 2, 2] = sols[:, 2], sols[:, 4], sols[:, 5]
    m = 0.5 * (m + np.transpose(m, (0, 2, 1)))
    evals, evecs = np.linalg.eigh(m)
    tr = (m[:, 0, 0] + m[:, 1, 1]) + m[:, 2, 2]
    ok = ~np.any(evals < (eig_floor * np.abs(tr))[:, None], axis=1)
    rq = np.stack([q / np.linalg.norm(q) for q in ref_quats]) if g else np.zeros((0, 4))
    ref = _quat_to_matrix_batch(rq)
    dots = np.abs(np.stack([ref[r].T @ evecs[r] for r in range(g)])) if g else np.zeros((0, 3, 3))
    sums = np.stack([((0 + dots[:, 0, p[0]]) + dots[:, 1, p[1]]) + dots[:, 2, p[2]]
                     for p in _PERMS], axis=1)
    best = np.asarray(_PERMS)[np.argmax(sums, axis=1)]  # first maximum, as max() over the list
    rows_ = np.arange(g)
    r = np.empty((g, 3, 3))
    scale = np.empty((g, 3))
    for k in range(3):
        e = evecs[rows_, :, best[:, k]]
        flip = np.array([np.dot(e[i], ref[i, :, k]) < 0 for i in range(g)], bool)
        e = np.where(flip[:, None], -e, e)
        r[:, :, k] = e
        scale[:, k] = np.sqrt(evals[rows_, best[:, k]])
    neg = np.linalg.det(r) < 0 if g else np.zeros(0, bool)
    r[neg, :, 2] = -r[neg, :, 2]
    q = np.empty((g, 4))
    for i in range(g):  # core.py:41-62 branches (scalar control flow, numpy arithmetic)
        q[i] = _matrix_to_quat(r[i])
    return q, scale, ok


def update_all(gaussians, motions, cameras, min_views=2, min_total_weight=1e-3,
               min_total_pixels=3, eig_floor=1e-12, loop=False):
    """multiview.py:168-275 over arrays.  Returns dict delta_mean (N,3), rotation (N,4),
    scale (N,3), status (N,) int8 and the eligibility mask.  `loop=True` runs the per-Gaussian
    loop of the reference verbatim; the default groups the LAPACK calls (same bits)."""
    g = _c(gaussians, np.float64).reshape(-1, 11)
    n = len(g)
    nv = len(cameras)
    means = g[:, 0:3].copy()
    quats = g[:, 3:7].copy()
    scales = g[:, 7:10].copy()
    rots = _quat_to_matrix_batch(quats)
    cov3 = rots * (scales ** 2)[:, None, :] @ np.transpose(rots, (0, 2, 1))

    solved = np.asarray(motions["status"]).reshape(nv, n) == STATUS_SOLVED
    weights = np.asarray(motions["weight_sum"], np.float64).reshape(nv, n)
    pixels = np.asarray(motions["pixel_count"]).reshape(nv, n).astype(np.int64)
    amot = np.asarray(motions["a"], np.float64).reshape(nv, n, 2, 2)
    bmot = np.asarray(motions["b"], np.float64).reshape(nv, n, 2)
    ok = np.zeros((nv, n), dtype=bool)
    rows = np.zeros((nv, n, 2, 4))
    lin = np.zeros((nv, n, 3, 6))
    rhs = np.zeros((nv, n, 3))
    for v, cam in enumerate(cameras):
        cam = np.asarray(cam, np.float64)
        rot = cam[:9].reshape(3, 3)
        trans = cam[9:12]
        fx, fy, cx, cy = cam[12], cam[13], cam[14], cam[15]
        a = amot[v]
        b = bmot[v]
        pc = means @ rot.T + trans
        z = pc[:, 2]
        in_front = z > 1e-6
        zs = np.where(in_front, z, 1.0)
        mean2 = np.stack([fx * pc[:, 0] / zs + cx, fy * pc[:, 1] / zs + cy], axis=1)
        j = np.zeros((n, 2, 3))
        j[:, 0, 0] = fx / zs
        j[:, 1, 1] = fy / zs
        j[:, 0, 2] = -fx * pc[:, 0] / (zs * zs)
        j[:, 1, 2] = -fy * pc[:, 1] / (zs * zs)
        m = j @ rot
        cov2 = m @ cov3 @ np.transpose(m, (0, 2, 1))
        cov2 = 0.5 * (cov2 + np.transpose(cov2, (0, 2, 1)))
        moved_mean = np.einsum("nij,nj->ni", a, mean2) + b
        moved_cov = a @ cov2 @ np.transpose(a, (0, 2, 1))
        moved_cov = 0.5 * (moved_cov + np.transpose(moved_cov, (0, 2, 1)))
        ok[v] = in_front & _min_eig_ok(cov2) & _min_eig_ok(moved_cov)
        p = _projection_matrix(cam)
        rows[v, :, 0] = moved_mean[:, 0, None] * p[2] - p[0]
        rows[v, :, 1] = moved_mean[:, 1, None] * p[2] - p[1]
        lin[v] = _vech_linearization(m)
        rhs[v] = np.stack([moved_cov[:, 0, 0], 0.5 * (moved_cov[:, 0, 1] + moved_cov[:, 1, 0]),
                           moved_cov[:, 1, 1]], axis=1)

    total_weight = np.where(solved, weights, 0.0).sum(axis=0)
    total_pixels = np.where(solved, pixels, 0).sum(axis=0)
    n_solved = solved.sum(axis=0)
    eligible = ((n_solved >= min_views) & (total_weight >= min_total_weight)
                & (total_pixels >= min_total_pixels) & ~np.any(solved & ~ok, axis=0))

    delta = np.zeros((n, 3))
    out_q = quats.copy()
    out_s = scales.copy()
    status = np.zeros(n, np.int8)
    fuse = _fuse_loop if loop else _fuse_batched
    fuse(np.flatnonzero(eligible), solved, rows, lin, rhs, means, quats, eig_floor, delta, out_q,
         out_s, status)
    return dict(delta_mean=delta, rotation=out_q, scale=out_s, status=status, eligible=eligible)


def _fuse_loop(idx, solved, rows, lin, rhs, means, quats, eig_floor, delta, out_q, out_s, status):
    """multiview.py:239-275, one Gaussian at a time (the reference's loop, verbatim order)."""
    with np.errstate(all="ignore"):
        for i in idx:
            sel = solved[:, i]
            a = rows[sel, i].reshape(-1, 4)
            try:
                _, s, vt = np.linalg.svd(a)
                if s[-2] - s[-1] <= _SINGULAR_GAP_REL * s[0]:
                    continue
                x = vt[-1]
                if abs(x[3]) <= _SINGULAR_GAP_REL * np.linalg.norm(x):
                    continue
                new_mean = x[:3] / x[3]
                u, s, vt = np.linalg.svd(lin[sel, i].reshape(-1, 6), full_matrices=False)
                if s[-1] < _SINGULAR_GAP_REL * s[0]:
                    continue
                sol = vt.T @ ((u.T @ rhs[sel, i].ravel()) / s)
                res = _decompose(sol, quats[i], eig_floor)
            except (np.linalg.LinAlgError, ValueError):
                continue
            if res is None:
                continue
            q, sc = res
            if not (np.all(np.isfinite(q)) and np.all(np.isfinite(new_mean)) and np.all(sc > 0)):
                continue
            delta[i] = new_mean - means[i]
            out_q[i] = q
            out_s[i] = sc
            status[i] = STATUS_SOLVED


def _fuse_batched(idx, solved, rows, lin, rhs, means, quats, eig_floor, delta, out_q, out_s,
                  status):
    """_fuse_loop over groups of Gaussians with the same solved-view count: the SVDs and eigh run
    as stacked LAPACK gufunc calls (per-matrix identical to the single calls); the few BLAS
    level-1/2 operations whose kernels may round differently when stacked (norm, dot, gemv) stay
    per Gaussian.  Bit-identical to _fuse_loop (tests/test_oracle_golden.py)."""
    if len(idx) == 0:
        return
    nsol = solved[:, idx].sum(axis=0)
    with np.errstate(all="ignore"):
        for k in np.unique(nsol):
            ids = idx[nsol == k]
            gi, vi = np.nonzero(solved[:, ids].T)  # per Gaussian, its solved views ascending
            a = rows[vi, ids[gi]].reshape(len(ids), 2 * k, 4)
            try:
                _, s, vt = np.linalg.svd(a)
            except np.linalg.LinAlgError:
                for j in ids:  # a failing stack: redo one by one (the loop's except path)
                    _fuse_loop(np.array([j]), solved, rows, lin, rhs, means, quats, eig_floor,
                               delta, out_q, out_s, status)
                continue
            ok = ~(s[:, -2] - s[:, -1] <= _SINGULAR_GAP_REL * s[:, 0])
            x = vt[:, -1]
            for r in np.flatnonzero(ok):
                if abs(x[r, 3]) <= _SINGULAR_GAP_REL * np.linalg.norm(x[r]):
                    ok[r] = False
            if not ok.any():
                continue
            sub = np.flatnonzero(ok)
            new_mean = x[sub, :3] / x[sub, 3:4]
            ids2 = ids[sub]
            lsel = lin[vi, ids[gi]].reshape(len(ids), 3 * k, 6)[sub]
            rsel = rhs[vi, ids[gi]].reshape(len(ids), 3 * k)[sub]
            try:
                u, s, vt = np.linalg.svd(lsel, full_matrices=False)
            except np.linalg.LinAlgError:
                for j in ids2:
                    _fuse_loop(np.array([j]), solved, rows, lin, rhs, means, quats, eig_floor,
                               delta, out_q, out_s, status)
                continue
            ok2 = np.flatnonzero(~(s[:, -1] < _SINGULAR_GAP_REL * s[:, 0]))
            if not len(ok2):
                continue
            sols = np.stack([vt[r].T @ ((u[r].T @ rsel[r]) / s[r]) for r in ok2])
            try:
                q, sc, ok3 = _decompose_batch(sols, quats[ids2[ok2]], eig_floor)
            except (np.linalg.LinAlgError, ValueError):
                for j in ids2[ok2]:
                    _fuse_loop(np.array([j]), solved, rows, lin, rhs, means, quats, eig_floor,
                               delta, out_q, out_s, status)
                continue
            nm = new_mean[ok2]
            good = (ok3 & np.all(np.isfinite(q), axis=1) & np.all(np.isfinite(nm), axis=1)
                    & np.all(sc > 0, axis=1))
            i = ids2[ok2[good]]
            delta[i] = nm[good] - means[i]
            out_q[i] = q[good]
            out_s[i] = sc[good]
            status[i] = STATUS_SOLVED


def compensate(gaussians, cameras, targets, valids, config=None):
    """The four hot-path stages of compensate_frame (pipeline.py:117-124 and :79-86), without
    regularisation.  targets: list of (H,W,2) f64; valids: list of (H,W) bool.
    Returns (updates, per-view motions list, per-view accumulators list)."""
    cfg = dict(alpha_cutoff=1.0 / 255.0, det_floor=1e-12, min_pixels=3, min_weight=1e-3,
               min_views=2, min_total_weight=1e-3, min_total_pixels=3, static_threshold_px=1.0,
               eig_floor=1e-12)
    if config:
        cfg.update(config)
    g = _c(gaussians, np.float64).reshape(-1, 11)
    n = len(g)
    accs, mots = [], []
    for cam, tgt, val in zip(cameras, targets, valids):
        wm = rasterize(g, cam, cfg["alpha_cutoff"])
        acc = accumulate(wm, tgt, val, n, cfg["static_threshold_px"])
        accs.append(acc)
        mots.append(solve_view(acc, cfg["det_floor"], cfg["min_pixels"], cfg["min_weight"]))
    stacked = {k: np.stack([m[k] for m in mots]) for k in ("status", "a", "b", "weight_sum",
                                                           "pixel_count")}
    upd = update_all(g, stacked, cameras, cfg["min_views"], cfg["min_total_weight"],
                     cfg["min_total_pixels"], cfg["eig_floor"])
    return upd, mots, accs


# ---------------------------------------------------------------------------
# oracle tracker (input production for the CPU arm and the tracker parity tests)

def relative_rotations(frame0, frame_t):
    """SceneSequence.relative_motion rotation for every Gaussian (scene.py:44-55):
    quat_to_matrix(g1.rotation) @ quat_to_matrix(g0.rotation).T, one 3x3 product per Gaussian
    as the reference forms it."""
    r0 = _quat_to_matrix_batch(np.asarray(frame0, np.float64)[:, 3:7])
    r1 = _quat_to_matrix_batch(np.asarray(frame_t, np.float64)[:, 3:7])
    return np.stack([r1[i] @ r0[i].T for i in range(len(r0))]) if len(r0) else r0


def dominant_gaussians(wm, width, height):
    """scene.py:166-189: per pixel the contribution with the largest alpha*T (ties by the smaller
    gaussian id).  Returns (gid (H,W) int64, -1 where empty; depth (H,W) float64)."""
    gid_img = np.full((height, width), -1, dtype=np.int64)
    depth_img = np.zeros((height, width))
    if len(wm["pixel_x"]) == 0:
        return gid_img, depth_img
    weight = wm["alpha"] * wm["transmittance"]
    pix = wm["pixel_y"].astype(np.int64) * width + wm["pixel_x"]
    order = np.lexsort((wm["gaussian_id"], -weight, pix))
    first = np.empty(len(order), dtype=bool)
    first[0] = True
    sorted_pix = pix[order]
    np.not_equal(sorted_pix[1:], sorted_pix[:-1], out=first[1:])
    sel = order[first]
    gid_img[wm["pixel_y"][sel], wm["pixel_x"][sel]] = wm["gaussian_id"][sel]
    depth_img[wm["pixel_y"][sel], wm["pixel_x"][sel]] = wm["depth"][sel]
    return gid_img, depth_img


def oracle_track(frame0, frame_t, camera, wm, view, target_frame, noise_sigma_px=0.0, seed=0,
                 rel=None):
    """scene.py:192-240 over arrays: every pixel back-projected onto the depth plane of its
    dominant Gaussian (from the frame-0 WeightMap `wm`), moved by that Gaussian's rigid motion
    frame0 -> frame_t and reprojected; keyed noise default_rng([seed, view, target_frame]).
    Returns (target (H,W,2) float64, valid (H,W) bool)."""
    cam = np.asarray(camera, np.float64)
    rot, trans = cam[:9].reshape(3, 3), cam[9:12]
    fx, fy, cx, cy = cam[12], cam[13], cam[14], cam[15]
    w, h = int(cam[16]), int(cam[17])
    gid_img, depth_img = dominant_gaussians(wm, w, h)
    valid = gid_img >= 0
    ys, xs = np.mgrid[0:h, 0:w]
    target = np.stack([xs, ys], axis=-1).astype(np.float64)
    vy, vx = np.nonzero(valid)
    if len(vy):
        f0 = np.asarray(frame0, np.float64)
        f1 = np.asarray(frame_t, np.float64)
        z = depth_img[vy, vx]
        pc = np.stack([(vx - cx) / fx * z, (vy - cy) / fy * z, z], axis=1)
        pw = (pc - trans) @ rot
        gids = gid_img[vy, vx]
        uniq, inv = np.unique(gids, return_inverse=True)
        rels = rel[uniq] if rel is not None else relative_rotations(f0[uniq], f1[uniq])
        mu0s = f0[uniq, 0:3]
        mu1s = f1[uniq, 0:3]
        moved = np.einsum("nij,nj->ni", rels[inv], pw - mu0s[inv]) + mu1s[inv]
        pc2 = moved @ rot.T + trans
        target[vy, vx, 0] = fx * pc2[:, 0] / pc2[:, 2] + cx
        target[vy, vx, 1] = fy * pc2[:, 1] / pc2[:, 2] + cy
    if noise_sigma_px > 0:
        rng = np.random.default_rng([seed, view, target_frame])
        noise = rng.normal(scale=noise_sigma_px, size=(h, w, 2))
        target[valid] += noise[valid]
    return target, valid
