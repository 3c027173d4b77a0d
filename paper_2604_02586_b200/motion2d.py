"""Per-view affine motion API (gausstrack/motion2d.py:20-204) backed by GPU kernels.

`accumulate_view` runs the deterministic segment-reduction kernel (bit-identical to np.add.at),
`solve_view` the batched 3x3 solve; `solve_view` returns a lazy `ViewMotionList` that behaves
like the reference's list of ViewMotion but only builds the Python objects that are touched.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .core import AffineMotion
from .errors import DimensionMismatch

DET_FLOOR_DEFAULT = 1e-12
MIN_PIXELS_DEFAULT = 3
MIN_WEIGHT_DEFAULT = 1e-3
STATIC_THRESHOLD_PX_DEFAULT = 1.0


class Status(enum.Enum):
    SOLVED = "solved"
    UNSOLVABLE = "unsolvable"
    STATIC = "static"


STATUS_CODE = {Status.UNSOLVABLE: 0, Status.SOLVED: 1, Status.STATIC: 2}
CODE_STATUS = {v: k for k, v in STATUS_CODE.items()}
_VALUE_CODE = {"unsolvable": 0, "solved": 1, "static": 2}


def status_code(status):
    """Integer status of a Status member -- ours or the reference's (matched by value, so
    gausstrack.motion2d.Status objects are accepted as well)."""
    return _VALUE_CODE.get(getattr(status, "value", status), 0)


@dataclass
class TrackField:
    """Dense per-view map from first-frame integer pixels to target positions."""

    view_id: int
    width: int
    height: int
    target: np.ndarray
    valid: np.ndarray

    def __post_init__(self):
        self.target = np.asarray(self.target, dtype=np.float64)
        self.valid = np.asarray(self.valid, dtype=bool)
        if self.target.shape != (self.height, self.width, 2):
            raise ValueError(f"target shape {self.target.shape} does not match "
                             f"{self.height}x{self.width}")
        if self.valid.shape != (self.height, self.width):
            raise ValueError("valid mask shape mismatch")
        if not np.all(np.isfinite(self.target[self.valid])):
            raise ValueError("valid track entries must be finite")

    @classmethod
    def identity(cls, view_id, width, height):
        ys, xs = np.mgrid[0:height, 0:width]
        return cls(view_id, width, height, np.stack([xs, ys], axis=-1).astype(np.float64),
                   np.ones((height, width), dtype=bool))


@dataclass
class MotionAccumulator:
    """Running weighted moments of one Gaussian in one view."""

    v1: np.ndarray = field(default_factory=lambda: np.zeros((3, 3)))
    v2: np.ndarray = field(default_factory=lambda: np.zeros((3, 2)))
    weight_sum: float = 0.0
    pixel_count: int = 0
    static_pixel_count: int = 0
    static_weight_sum: float = 0.0


@dataclass
class ViewMotion:
    gaussian_id: int
    view_id: int
    motion: AffineMotion
    weight_sum: float
    pixel_count: int
    status: Status


@dataclass
class ViewAccumulators:
    """Per-Gaussian moment arrays of one view."""

    view_id: int
    v1: np.ndarray
    v2: np.ndarray
    weight_sum: np.ndarray
    pixel_count: np.ndarray
    static_pixel_count: np.ndarray
    static_weight_sum: np.ndarray


class ViewMotionList:
    """Array-backed, lazily materialised list[ViewMotion] of one view."""

    def __init__(self, view_id, status, a, b, weight_sum, pixel_count):
        self.view_id = view_id
        self.status = np.asarray(status, np.int8)
        self.a = np.asarray(a, np.float64).reshape(-1, 2, 2)
        self.b = np.asarray(b, np.float64).reshape(-1, 2)
        self.weight_sum = np.asarray(weight_sum, np.float64)
        self.pixel_count = np.asarray(pixel_count, np.int64)

    def __len__(self):
        return len(self.status)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        solved = self.status[i] == 1
        motion = AffineMotion(self.a[i], self.b[i]) if solved else AffineMotion.identity()
        return ViewMotion(i, self.view_id, motion, float(self.weight_sum[i]),
                          int(self.pixel_count[i]), Status.SOLVED if solved else Status.UNSOLVABLE)

    def __iter__(self):
        return (self[i] for i in range(len(self)))


def motions_arrays(vms):
    """(status, a, b, weight_sum, pixel_count) arrays of a ViewMotionList or list[ViewMotion]."""
    if isinstance(vms, ViewMotionList):
        return vms.status, vms.a, vms.b, vms.weight_sum, vms.pixel_count
    n = len(vms)
    status = np.array([status_code(vm.status) for vm in vms], np.int8).reshape(n)
    a = np.array([vm.motion.a for vm in vms], np.float64).reshape(n, 2, 2)
    b = np.array([vm.motion.b for vm in vms], np.float64).reshape(n, 2)
    w = np.array([vm.weight_sum for vm in vms], np.float64).reshape(n)
    c = np.array([vm.pixel_count for vm in vms], np.int64).reshape(n)
    return status, a, b, w, c


def accumulate(acc: MotionAccumulator, x, x_prime, w,
               static_threshold_px=STATIC_THRESHOLD_PX_DEFAULT) -> MotionAccumulator:
    """Scalar running update with one weighted correspondence (host-side bookkeeping; the
    batched equivalent is `accumulate_view`)."""
    x = np.asarray(x, dtype=np.float64)
    xp = np.asarray(x_prime, dtype=np.float64)
    h = np.array([x[0], x[1], 1.0])
    acc.v1 += w * np.outer(h, h)
    acc.v2 += w * np.outer(h, xp)
    acc.weight_sum += w
    acc.pixel_count += 1
    if np.linalg.norm(xp - x) < static_threshold_px:
        acc.static_pixel_count += 1
        acc.static_weight_sum += w
    return acc


def _solve_arrays(v1, v2, wsum, cnt, det_floor, min_pixels, min_weight):
    import torch

    from .engine import as_device
    n = len(wsum)
    lib = nat.lib()
    f64 = torch.float64
    dv1 = as_device(np.asarray(v1, np.float64).reshape(n, 9), f64)
    dv2 = as_device(np.asarray(v2, np.float64).reshape(n, 6), f64)
    dw = as_device(np.asarray(wsum, np.float64).reshape(n), f64)
    dc = as_device(np.asarray(cnt, np.int64).reshape(n), torch.int64)
    st = torch.empty(n, dtype=torch.int8, device=dv1.device)
    a = torch.empty((n, 2, 2), dtype=f64, device=dv1.device)
    b = torch.empty((n, 2), dtype=f64, device=dv1.device)
    nat.check(lib.ts_solve_view(nat.dptr(dv1), nat.dptr(dv2), nat.dptr(dw), nat.dptr(dc), n,
                                float(det_floor), int(min_pixels), float(min_weight),
                                nat.dptr(st), nat.dptr(a), nat.dptr(b), None, nat.stream_ptr()),
              "solve_view")
    return st.cpu().numpy(), a.cpu().numpy(), b.cpu().numpy()


def solve_motion(acc: MotionAccumulator, det_floor=DET_FLOOR_DEFAULT,
                 min_pixels=MIN_PIXELS_DEFAULT, min_weight=MIN_WEIGHT_DEFAULT, gaussian_id=-1,
                 view_id=-1) -> ViewMotion:
    """[A|b] of one accumulator (K3 with batch 1); degeneracy gives UNSOLVABLE."""
    st, a, b = _solve_arrays(acc.v1[None], acc.v2[None], [acc.weight_sum], [acc.pixel_count],
                             det_floor, min_pixels, min_weight)
    if st[0] == 1:
        return ViewMotion(gaussian_id, view_id, AffineMotion(a[0], b[0]), acc.weight_sum,
                          acc.pixel_count, Status.SOLVED)
    return ViewMotion(gaussian_id, view_id, AffineMotion.identity(), acc.weight_sum,
                      acc.pixel_count, Status.UNSOLVABLE)


def accumulate_view(weightmap, track: TrackField, n_gaussians: int,
                    static_threshold_px=STATIC_THRESHOLD_PX_DEFAULT) -> ViewAccumulators:
    """All contributions with a valid track into per-Gaussian moments, on the GPU, in
    contribution order (bit-identical to the reference's np.add.at)."""
    import torch

    from .engine import as_device
    if (weightmap.width, weightmap.height) != (track.width, track.height):
        raise DimensionMismatch(f"weight map {weightmap.width}x{weightmap.height} vs "
                                f"track field {track.width}x{track.height}")
    n = int(n_gaussians)
    m = len(weightmap)
    gid_host = np.asarray(weightmap.gaussian_id, np.int64)
    if m and (gid_host.min() < 0 or gid_host.max() >= n):
        raise IndexError("gaussian_id out of range for n_gaussians")
    lib = nat.lib()
    plan = nat.default_plan()
    f64 = torch.float64
    px = as_device(np.asarray(weightmap.pixel_x, np.int32), torch.int32)
    py = as_device(np.asarray(weightmap.pixel_y, np.int32), torch.int32)
    gid = as_device(gid_host, torch.int64)
    al = as_device(np.asarray(weightmap.alpha, np.float64), f64)
    tr = as_device(np.asarray(weightmap.transmittance, np.float64), f64)
    tgt = as_device(track.target, f64)
    val = as_device(track.valid.astype(np.uint8), torch.uint8)
    dev = tgt.device
    v1 = torch.empty((n, 3, 3), dtype=f64, device=dev)
    v2 = torch.empty((n, 3, 2), dtype=f64, device=dev)
    ws = torch.empty(n, dtype=f64, device=dev)
    cnt = torch.empty(n, dtype=torch.int64, device=dev)
    scnt = torch.empty(n, dtype=torch.int64, device=dev)
    sws = torch.empty(n, dtype=f64, device=dev)
    nat.check(lib.ts_accumulate_view(plan.handle, nat.dptr(px), nat.dptr(py), nat.dptr(gid),
                                     nat.dptr(al), nat.dptr(tr), m, int(track.width),
                                     int(track.height), nat.dptr(tgt), nat.TS_TRACK_F64,
                                     nat.dptr(val), n, float(static_threshold_px), nat.dptr(v1),
                                     nat.dptr(v2), nat.dptr(ws), nat.dptr(cnt), nat.dptr(scnt),
                                     nat.dptr(sws), nat.stream_ptr()), "accumulate_view")
    return ViewAccumulators(weightmap.view_id, v1.cpu().numpy(), v2.cpu().numpy(),
                            ws.cpu().numpy(), cnt.cpu().numpy(), scnt.cpu().numpy(),
                            sws.cpu().numpy())


def solve_view(acc: ViewAccumulators, det_floor=DET_FLOOR_DEFAULT,
               min_pixels=MIN_PIXELS_DEFAULT, min_weight=MIN_WEIGHT_DEFAULT):
    """Every Gaussian's motion in one view (GPU), as a lazy list of ViewMotion."""
    n = len(acc.weight_sum)
    if n == 0:
        return ViewMotionList(acc.view_id, np.empty(0), np.empty((0, 2, 2)), np.empty((0, 2)),
                              np.empty(0), np.empty(0))
    st, a, b = _solve_arrays(acc.v1, acc.v2, acc.weight_sum, acc.pixel_count, det_floor,
                             min_pixels, min_weight)
    return ViewMotionList(acc.view_id, st, a, b, acc.weight_sum, acc.pixel_count)


def solve_all_views(weightmaps, tracks, n_gaussians, det_floor=DET_FLOOR_DEFAULT,
                    min_pixels=MIN_PIXELS_DEFAULT, min_weight=MIN_WEIGHT_DEFAULT,
                    static_threshold_px=STATIC_THRESHOLD_PX_DEFAULT):
    """accumulate_view + solve_view per view; returns (motions, accumulators)."""
    if len(weightmaps) != len(tracks):
        raise DimensionMismatch("weight maps and track fields count differ")
    motions, accs = [], []
    for wm, tf in zip(weightmaps, tracks):
        acc = accumulate_view(wm, tf, n_gaussians, static_threshold_px)
        accs.append(acc)
        motions.append(solve_view(acc, det_floor, min_pixels, min_weight))
    return motions, accs
