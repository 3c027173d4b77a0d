"""Motion regularisation on the GPU (gausstrack/regularize.py:37-188).

Same public names and semantics as the reference module -- exact kNN with (distance, id) ties,
static detection, componentwise median filter with polar projection, propagation with an
intrinsic-XYZ Euler circular mean, apply_updates -- backed by csrc/regularize.cu through the C
ABI (ts_build_knn, ts_detect_static, ts_median_filter, ts_propagate, ts_apply_updates,
ts_regularize).  `regularize_device` is the tensor-native form used by `compensate_frame`
(the _fuse_frame tail, pipeline.py:88-98): two kernels after K4, no host round trip.

kNN parity is bit-exact (distances are formed like numpy's norm); the rotation stages are
floating-point restatements of LAPACK / scipy / libm calls and agree to ~1e-12
(tests/test_gpu_regularize.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import Gaussian3D, gaussians_array
from .motion2d import Status, status_code
from .multiview import MotionUpdate

KNN_K_DEFAULT = 8
MIN_HIT_PIXELS_DEFAULT = 9
STATIC_FRACTION_DEFAULT = 0.9
STATIC_MIN_VIEWS_DEFAULT = 2
SCALE_CLAMP = 1e-9

_STATUS = {0: Status.UNSOLVABLE, 1: Status.SOLVED, 2: Status.STATIC}


@dataclass(frozen=True)
class StaticStats:
    """Per-view (pixel_count, static_pixel_count) tallies for one Gaussian."""

    gaussian_id: int
    per_view: tuple


@dataclass(frozen=True)
class NeighborIndex:
    positions: np.ndarray  # (N, 3)
    k: int
    adjacency: np.ndarray  # (N, min(k, N-1)) int64


def _torch():
    import torch
    return torch


def _dev(x, dtype):
    from .engine import as_device
    return as_device(x, dtype)


def _updates_struct(delta, rot, scale, status):
    return nat.Updates(nat.dptr(delta).value, nat.dptr(rot).value, nat.dptr(scale).value,
                       nat.dptr(status).value)


def _empty_updates(n, device):
    torch = _torch()
    f64 = dict(dtype=torch.float64, device=device)
    return (torch.empty((n, 3), **f64), torch.empty((n, 4), **f64), torch.empty((n, 3), **f64),
            torch.empty(n, dtype=torch.int8, device=device))


# -- tensor-native entry points -----------------------------------------------------------------

def knn_device(positions, k=KNN_K_DEFAULT, plan=None, stream=None):
    """(N, min(k, N-1)) int64 CUDA adjacency of an (N, 3) positions tensor or (N, 11) rows."""
    torch = _torch()
    pos = positions if isinstance(positions, torch.Tensor) else np.asarray(positions, np.float64)
    pos = _dev(pos, torch.float64)
    if pos.dim() != 2 or pos.shape[1] not in (3, 11):
        raise ValueError("positions must be (N, 3) or Gaussian rows (N, 11)")
    n = int(pos.shape[0])
    if n < 2:
        raise ValueError("need at least 2 positions")
    kk = min(int(k), n - 1)
    if kk < 1 or kk > nat.TS_KNN_MAX_K:
        raise ValueError(f"k must be in [1, {nat.TS_KNN_MAX_K}], got {k}")
    adj = torch.empty((n, kk), dtype=torch.int64, device=pos.device)
    plan = plan if plan is not None else nat.default_plan()
    nat.check(nat.lib().ts_build_knn(plan.handle, nat.dptr(pos), int(pos.shape[1]), n, kk,
                                     nat.dptr(adj), nat.stream_ptr(stream)), "ts_build_knn")
    return adj


def regularize_device(frame1, delta, rotation, scale, status, pixel_count, static_pixel_count,
                      n_views, adjacency, config=None, plan=None, stream=None):
    """The _fuse_frame regularisation tail (pipeline.py:88-98) on device tensors.

    frame1 (N, 11) f64; K4 updates delta (N,3), rotation (N,4), scale (N,3), status (N,) int8;
    counts (V*N,) int32 view-major; adjacency (N, kk) int64.  Returns
    (delta, rotation, scale, status, static_flags, rows) -- new tensors, inputs untouched.
    """
    torch = _torch()
    n = int(frame1.shape[0])
    out = _empty_updates(n, frame1.device)
    flags = torch.empty(n, dtype=torch.uint8, device=frame1.device)
    rows = torch.empty((n, 11), dtype=torch.float64, device=frame1.device)
    cfg = nat.make_reg_config(config)
    uin = _updates_struct(delta, rotation, scale, status)
    uout = _updates_struct(*out)
    plan = plan if plan is not None else nat.default_plan()
    kk = int(adjacency.shape[1]) if adjacency is not None and adjacency.dim() == 2 else 0
    nat.check(nat.lib().ts_regularize(plan.handle, nat.dptr(frame1), n, ctypes.byref(uin),
                                      nat.dptr(pixel_count), nat.dptr(static_pixel_count),
                                      int(n_views), nat.dptr(adjacency), kk, ctypes.byref(cfg),
                                      ctypes.byref(uout), nat.dptr(flags), nat.dptr(rows),
                                      nat.stream_ptr(stream)), "ts_regularize")
    return out + (flags, rows)


def apply_rows_device(frame1, delta, rotation, scale, status, stream=None):
    """apply_updates (regularize.py:177-188) on device tensors -> (N, 11) rows."""
    torch = _torch()
    n = int(frame1.shape[0])
    rows = torch.empty((n, 11), dtype=torch.float64, device=frame1.device)
    u = _updates_struct(delta, rotation, scale, status)
    nat.check(nat.lib().ts_apply_updates(nat.dptr(frame1), n, ctypes.byref(u), nat.dptr(rows),
                                         nat.stream_ptr(stream)), "ts_apply_updates")
    return rows


# -- reference-typed API ------------------------------------------------------------------------

def build_knn(positions, k=KNN_K_DEFAULT) -> NeighborIndex:
    """Exact k-nearest neighbours by Euclidean distance, ties by ascending id (GPU grid search)."""
    positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    if len(positions) < 2:
        raise ValueError("need at least 2 positions")
    adj = knn_device(positions, k)
    return NeighborIndex(positions, k, adj.cpu().numpy())


def detect_static_all(pixel_counts, static_counts, min_hit_pixels=MIN_HIT_PIXELS_DEFAULT,
                      static_fraction=STATIC_FRACTION_DEFAULT,
                      min_views=STATIC_MIN_VIEWS_DEFAULT):
    """Static flags from (G, V) count arrays (regularize.py:77-88)."""
    torch = _torch()
    pc = np.asarray(pixel_counts).reshape(len(pixel_counts), -1)
    sc = np.asarray(static_counts).reshape(pc.shape)
    g, v = pc.shape
    if g == 0:
        return np.zeros(0, bool)
    dpc = _dev(np.ascontiguousarray(pc.T).astype(np.int32), torch.int32)
    dsc = _dev(np.ascontiguousarray(sc.T).astype(np.int32), torch.int32)
    flags = torch.empty(g, dtype=torch.uint8, device=dpc.device)
    cfg = nat.RegConfig()
    cfg.min_hit_pixels, cfg.min_views = int(min_hit_pixels), int(min_views)
    cfg.static_fraction = float(static_fraction)
    nat.check(nat.lib().ts_detect_static(nat.dptr(dpc), nat.dptr(dsc), g, v, ctypes.byref(cfg),
                                         nat.dptr(flags), nat.stream_ptr()), "ts_detect_static")
    return flags.cpu().numpy().astype(bool)


def detect_static(stats: StaticStats, min_hit_pixels=MIN_HIT_PIXELS_DEFAULT,
                  static_fraction=STATIC_FRACTION_DEFAULT,
                  min_views=STATIC_MIN_VIEWS_DEFAULT) -> bool:
    """True iff at least `min_views` views have pixel_count > min_hit_pixels and
    static_pixel_count > static_fraction * pixel_count (strict, regularize.py:56-74)."""
    pv = np.array(stats.per_view, dtype=np.int64).reshape(1, -1, 2)
    return bool(detect_static_all(pv[..., 0], pv[..., 1], min_hit_pixels, static_fraction,
                                  min_views)[0])


def updates_arrays(updates):
    """(delta (N,3), rotation (N,4), scale (N,3), status (N,) int8) of a list of MotionUpdate."""
    if hasattr(updates, "delta_mean") and hasattr(updates, "status") and \
            not isinstance(updates, MotionUpdate):
        return (updates.delta_mean, updates.rotation, updates.scale,
                np.asarray(updates.status, np.int8))
    n = len(updates)
    d = np.array([u.delta_mean for u in updates], np.float64).reshape(n, 3)
    q = np.array([u.new_rotation for u in updates], np.float64).reshape(n, 4)
    s = np.array([u.new_scale for u in updates], np.float64).reshape(n, 3)
    st = np.array([status_code(u.status) for u in updates], np.int8)
    return d, q, s, st


def _device_updates(updates):
    torch = _torch()
    d, q, s, st = updates_arrays(updates)
    f64 = torch.float64
    return _dev(d, f64), _dev(q, f64), _dev(s, f64), _dev(st, torch.int8)


def _gid(u, i):
    return getattr(u, "gaussian_id", i)


def _materialise(updates, out, changed):
    d, q, s, st = (t.cpu().numpy() for t in out)
    res = list(updates)
    for i in np.flatnonzero(changed):
        res[i] = MotionUpdate(_gid(updates[i], i), d[i].copy(), q[i].copy(), s[i].copy(),
                              _STATUS[int(st[i])])
    return res


def _adjacency(index: NeighborIndex):
    torch = _torch()
    adj = np.asarray(index.adjacency, np.int64)
    return _dev(adj.reshape(len(adj), -1), torch.int64)


def median_filter(updates, index: NeighborIndex, frame1) -> list:
    """Replace each solved Gaussian's deltas by the componentwise median over itself and its
    solved neighbours; rotations are projected back with the polar factor (regularize.py:91-121).
    Non-solved entries pass through as the same objects."""
    rows = gaussians_array(frame1)
    g = _dev(rows, _torch().float64)
    uin = _device_updates(updates)
    out = _empty_updates(len(rows), g.device)
    adj = _adjacency(index)
    nat.check(nat.lib().ts_median_filter(nat.dptr(g), len(rows),
                                         ctypes.byref(_updates_struct(*uin)), nat.dptr(adj),
                                         int(adj.shape[1]), ctypes.byref(_updates_struct(*out)),
                                         nat.stream_ptr()), "ts_median_filter")
    return _materialise(updates, out, uin[3].cpu().numpy() == 1)


def propagate(updates, index: NeighborIndex, static_flags, frame1, average="mean") -> list:
    """Pin static Gaussians to frame 1 and fill unsolvable ones from solved, non-static
    neighbours (regularize.py:124-174)."""
    if average not in ("mean", "median"):
        raise ValueError(f"average must be 'mean' or 'median', got {average}")
    torch = _torch()
    rows = gaussians_array(frame1)
    g = _dev(rows, torch.float64)
    uin = _device_updates(updates)
    out = _empty_updates(len(rows), g.device)
    adj = _adjacency(index)
    flags = _dev(np.asarray(static_flags, bool).astype(np.uint8), torch.uint8)
    nat.check(nat.lib().ts_propagate(nat.default_plan().handle, nat.dptr(g), len(rows),
                                     ctypes.byref(_updates_struct(*uin)), nat.dptr(adj),
                                     int(adj.shape[1]), nat.dptr(flags),
                                     0 if average == "mean" else 1,
                                     ctypes.byref(_updates_struct(*out)), nat.stream_ptr()),
              "ts_propagate")
    before = uin[3].cpu().numpy()
    after = out[3].cpu().numpy()
    changed = np.asarray(static_flags, bool) | (before != after)
    return _materialise(updates, out, changed)


def apply_updates(frame1, updates) -> list:
    """Updated Gaussians; unsolvable entries keep the frame-1 objects (regularize.py:177-188)."""
    rows = gaussians_array(frame1)
    g = _dev(rows, _torch().float64)
    u = _device_updates(updates)
    out = _torch().empty((len(rows), 11), dtype=_torch().float64, device=g.device)
    nat.check(nat.lib().ts_apply_updates(nat.dptr(g), len(rows), ctypes.byref(_updates_struct(*u)),
                                         nat.dptr(out), nat.stream_ptr()), "ts_apply_updates")
    new = out.cpu().numpy()
    q = u[1].cpu().numpy()
    st = u[3].cpu().numpy()
    res = []
    for i in range(len(rows)):
        if st[i] == 0:
            res.append(frame1[i])
        else:  # Gaussian3D normalises the update's quaternion itself (core.py:95-106)
            r = new[i]
            res.append(Gaussian3D(r[0:3], q[i], r[7:10], r[10]))
    return res
