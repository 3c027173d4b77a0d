"""Multi-view fuse API (gausstrack/multiview.py:24-315) backed by K4 on the GPU.

`update_all` runs the fused kernel (one thread per Gaussian, streaming QR + Jacobi solves in
registers) and returns a lazy `MotionUpdateList`.  The scalar KAT entry points
(`triangulate_mean`, `solve_covariance3d`, `decompose_covariance`, `update_gaussian`) call the same
device routines with a batch of one, raising the reference's exceptions on failure.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import Gaussian2D, Sym3, cameras_array, gaussians_array
from .errors import (DegenerateGeometry, InsufficientViews, NegativeEigenvalue,
                     RankDeficient)
from .motion2d import Status, motions_arrays, status_code

MIN_VIEWS_DEFAULT = 2
MIN_TOTAL_WEIGHT_DEFAULT = 1e-3
MIN_TOTAL_PIXELS_DEFAULT = 3
EIG_FLOOR_DEFAULT = 1e-12
_SINGULAR_GAP_REL = 1e-9


@dataclass(frozen=True)
class ViewObservation:
    view_id: int
    updated: Gaussian2D
    linearization: np.ndarray
    weight_sum: float


@dataclass
class MotionUpdate:
    gaussian_id: int
    delta_mean: np.ndarray
    new_rotation: np.ndarray
    new_scale: np.ndarray
    status: Status


class MotionUpdateList:
    """Array-backed, lazily materialised list[MotionUpdate]."""

    def __init__(self, delta_mean, rotation, scale, status):
        self.delta_mean = np.asarray(delta_mean, np.float64).reshape(-1, 3)
        self.rotation = np.asarray(rotation, np.float64).reshape(-1, 4)
        self.scale = np.asarray(scale, np.float64).reshape(-1, 3)
        self.status = np.asarray(status, np.int8)

    def __len__(self):
        return len(self.status)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        st = {0: Status.UNSOLVABLE, 1: Status.SOLVED, 2: Status.STATIC}[int(self.status[i])]
        return MotionUpdate(i, self.delta_mean[i].copy(), self.rotation[i].copy(),
                            self.scale[i].copy(), st)

    def __iter__(self):
        return (self[i] for i in range(len(self)))


def _dev(x, dtype):
    from .engine import as_device
    return as_device(x, dtype)


def triangulate_mean(observations):
    """Homogeneous DLT triangulation of (CameraView, pixel mean) pairs (GPU QR + Jacobi SVD)."""
    import torch
    if len(observations) < 2:
        raise InsufficientViews(f"need >= 2 views, got {len(observations)}")
    rows = []
    for view, mean2 in observations:
        p = view.projection_matrix()
        u, v = np.asarray(mean2, dtype=np.float64)
        rows.append(u * p[2] - p[0])
        rows.append(v * p[2] - p[1])
    a = np.stack(rows)[None]
    x = torch.empty((1, 3), dtype=torch.float64, device="cuda")
    st = torch.empty(1, dtype=torch.int8, device="cuda")
    nr = _dev(np.array([len(rows)], np.int32), torch.int32)
    da = _dev(a, torch.float64)  # keep alive until the launch is enqueued
    nat.check(nat.lib().ts_triangulate_batch(nat.dptr(da), nat.dptr(nr), 1,
                                             len(rows), nat.dptr(x), nat.dptr(st),
                                             nat.stream_ptr()), "triangulate")
    if int(st[0]) != 1:
        raise DegenerateGeometry("triangulation system has no unique solution")
    return x[0].cpu().numpy()


_VECH_IJ = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]


def _vech_block(m):
    m0, m1 = m[0], m[1]
    cols = []
    for i, j in _VECH_IJ:
        if i == j:
            cols.append([m0[i] * m0[i], m0[i] * m1[i], m1[i] * m1[i]])
        else:
            cols.append([2.0 * m0[i] * m0[j], m0[i] * m1[j] + m0[j] * m1[i],
                         2.0 * m1[i] * m1[j]])
    return np.array(cols).T


def solve_covariance3d(observations) -> Sym3:
    """Least-squares 3D covariance from (M, cov2) pairs (GPU QR + Jacobi rank test)."""
    import torch
    if len(observations) < 2:
        raise InsufficientViews(f"need >= 2 views, got {len(observations)}")
    blocks, rhs = [], []
    for m, cov2 in observations:
        m = np.asarray(m, dtype=np.float64)
        c = np.asarray(cov2, dtype=np.float64)
        blocks.append(_vech_block(m))
        rhs.append([c[0, 0], 0.5 * (c[0, 1] + c[1, 0]), c[1, 1]])
    lin = np.concatenate(blocks)[None]
    b = np.concatenate(rhs)[None]
    x = torch.empty((1, 6), dtype=torch.float64, device="cuda")
    st = torch.empty(1, dtype=torch.int8, device="cuda")
    nr = _dev(np.array([lin.shape[1]], np.int32), torch.int32)
    dl, db = _dev(lin, torch.float64), _dev(b, torch.float64)
    nat.check(nat.lib().ts_solve_cov3d_batch(nat.dptr(dl), nat.dptr(db), nat.dptr(nr), 1,
                                             lin.shape[1], nat.dptr(x), nat.dptr(st),
                                             nat.stream_ptr()), "solve_covariance3d")
    if int(st[0]) != 1:
        raise RankDeficient("stacked system rank deficient")
    return Sym3(*[float(v) for v in x[0].cpu().numpy()])


def decompose_covariance(sigma, reference_rotation, reference_scale,
                         eig_floor=EIG_FLOOR_DEFAULT):
    """(quaternion, scale) of a 3D covariance with eigenpairs matched to the reference axes."""
    import torch
    m = sigma.matrix if isinstance(sigma, Sym3) else np.asarray(sigma, dtype=np.float64)
    q = torch.empty((1, 4), dtype=torch.float64, device="cuda")
    s = torch.empty((1, 3), dtype=torch.float64, device="cuda")
    st = torch.empty(1, dtype=torch.int8, device="cuda")
    ref = np.asarray(reference_rotation, np.float64).reshape(1, 4)
    dm, dr = _dev(m.reshape(1, 3, 3), torch.float64), _dev(ref, torch.float64)
    nat.check(nat.lib().ts_decompose_batch(nat.dptr(dm), nat.dptr(dr), 1,
                                           float(eig_floor), nat.dptr(q), nat.dptr(s),
                                           nat.dptr(st), nat.stream_ptr()), "decompose")
    if int(st[0]) != 1:
        raise NegativeEigenvalue("eigenvalue below floor")
    return q[0].cpu().numpy(), s[0].cpu().numpy()


def update_arrays(gaussians_rows, cameras, status, a, b, weight_sum, pixel_count, config=None,
                  **thresholds):
    """K4 over SoA inputs; returns (delta (N,3), rotation (N,4), scale (N,3), status (N,))."""
    import torch

    from .config import Config
    rows = gaussians_array(gaussians_rows)
    n = len(rows)
    cams = cameras_array(cameras)
    nv = len(cams)
    cfg = nat.make_config(config if config is not None else Config(**thresholds)
                          if thresholds else None)
    f64 = torch.float64
    g = _dev(rows, f64)
    st = _dev(np.asarray(status, np.int8).reshape(nv * n), torch.int8)
    da = _dev(np.asarray(a, np.float64).reshape(nv * n, 4), f64)
    db = _dev(np.asarray(b, np.float64).reshape(nv * n, 2), f64)
    dw = _dev(np.asarray(weight_sum, np.float64).reshape(nv * n), f64)
    dc = _dev(np.asarray(pixel_count).reshape(nv * n).astype(np.int32), torch.int32)
    dev = g.device
    out_d = torch.empty((n, 3), dtype=f64, device=dev)
    out_q = torch.empty((n, 4), dtype=f64, device=dev)
    out_s = torch.empty((n, 3), dtype=f64, device=dev)
    out_st = torch.empty(n, dtype=torch.int8, device=dev)
    m = nat.Motions(nat.dptr(st).value, nat.dptr(da).value, nat.dptr(db).value,
                    nat.dptr(dw).value, nat.dptr(dc).value, None, None)
    u = nat.Updates(nat.dptr(out_d).value, nat.dptr(out_q).value, nat.dptr(out_s).value,
                    nat.dptr(out_st).value)
    nat.check(nat.lib().ts_update_all(nat.dptr(g), n, nat.make_cameras(cams), nv,
                                      ctypes.byref(m), ctypes.byref(cfg), ctypes.byref(u),
                                      nat.stream_ptr()), "update_all")
    return (out_d.cpu().numpy(), out_q.cpu().numpy(), out_s.cpu().numpy(),
            out_st.cpu().numpy())


def update_all(gaussians, motions, views, min_views=MIN_VIEWS_DEFAULT,
               min_total_weight=MIN_TOTAL_WEIGHT_DEFAULT,
               min_total_pixels=MIN_TOTAL_PIXELS_DEFAULT, eig_floor=EIG_FLOOR_DEFAULT):
    """Fuse per-view motions of every Gaussian (K4); lazy list[MotionUpdate]."""
    rows = gaussians_array(gaussians)
    parts = [motions_arrays(vms) for vms in motions]
    n = len(rows)
    nv = len(views)
    st = np.stack([p[0] for p in parts]).reshape(nv, n)
    a = np.stack([p[1] for p in parts]).reshape(nv, n, 2, 2)
    b = np.stack([p[2] for p in parts]).reshape(nv, n, 2)
    w = np.stack([p[3] for p in parts]).reshape(nv, n)
    c = np.stack([p[4] for p in parts]).reshape(nv, n)
    d, q, s, ust = update_arrays(rows, views, st, a, b, w, c, min_views=min_views,
                                 min_total_weight=min_total_weight,
                                 min_total_pixels=min_total_pixels, eig_floor=eig_floor)
    return MotionUpdateList(d, q, s, ust)


def update_gaussian(g, view_motions, views, gaussian_id=-1, min_views=MIN_VIEWS_DEFAULT,
                    min_total_weight=MIN_TOTAL_WEIGHT_DEFAULT,
                    min_total_pixels=MIN_TOTAL_PIXELS_DEFAULT,
                    eig_floor=EIG_FLOOR_DEFAULT) -> MotionUpdate:
    """Fuse one Gaussian's view motions (K4 with N = 1)."""
    nv = len(views)
    st = np.zeros((nv, 1), np.int8)
    a = np.tile(np.eye(2), (nv, 1, 1, 1))
    b = np.zeros((nv, 1, 2))
    w = np.zeros((nv, 1))
    c = np.zeros((nv, 1), np.int64)
    for vm in view_motions:
        if status_code(vm.status) != 1:
            continue
        v = vm.view_id
        st[v, 0] = 1
        a[v, 0] = vm.motion.a
        b[v, 0] = vm.motion.b
        w[v, 0] = vm.weight_sum
        c[v, 0] = vm.pixel_count
    d, q, s, ust = update_arrays([g], views, st, a, b, w, c, min_views=min_views,
                                 min_total_weight=min_total_weight,
                                 min_total_pixels=min_total_pixels, eig_floor=eig_floor)
    if ust[0] == 1:
        return MotionUpdate(gaussian_id, d[0], q[0], s[0], Status.SOLVED)
    return MotionUpdate(gaussian_id, np.zeros(3), g.rotation.copy(), g.scale.copy(),
                        Status.UNSOLVABLE)
