"""Weight rasterizer API (gausstrack/splat.py:17-195) backed by K1 + K2 on the GPU.

`rasterize_weights` keeps the reference signature and returns the same `WeightMap` (host numpy
arrays in the reference order: pixel row-major, then depth, then Gaussian id).  On the device it
runs the fused raster kernel in contribution-emitting mode; the fused hot path
(`engine.FrameEngine`) never materialises weight maps.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import DegenerateCovariance

ALPHA_CUTOFF_DEFAULT = 1.0 / 255.0
ALPHA_CLAMP = 0.999
EARLY_STOP_TRANSMITTANCE = 1e-4
DET_FLOOR = 1e-12
SIGMA_RADIUS = 3.0


@dataclass(frozen=True)
class PixelContribution:
    gaussian_id: int
    pixel: tuple
    alpha: float
    transmittance: float


@dataclass
class WeightMap:
    """Surviving per-pixel contributions of one view, as parallel arrays sorted by pixel
    (row-major), then front-to-back depth, ties by Gaussian id."""

    view_id: int
    width: int
    height: int
    pixel_x: np.ndarray
    pixel_y: np.ndarray
    gaussian_id: np.ndarray
    alpha: np.ndarray
    transmittance: np.ndarray
    depth: np.ndarray
    degenerate_ids: list = field(default_factory=list)

    def __len__(self):
        return len(self.gaussian_id)

    def contributions(self):
        for k in range(len(self)):
            yield PixelContribution(int(self.gaussian_id[k]),
                                    (int(self.pixel_x[k]), int(self.pixel_y[k])),
                                    float(self.alpha[k]), float(self.transmittance[k]))

    def dump(self, path):
        """One line per contribution: view px py gid alpha transmittance."""
        with open(path, "w") as fh:
            for k in range(len(self)):
                fh.write(f"{self.view_id} {self.pixel_x[k]} {self.pixel_y[k]} "
                         f"{self.gaussian_id[k]} {self.alpha[k]:.9g} "
                         f"{self.transmittance[k]:.9g}\n")


def invert_2x2(cov2, det_floor=DET_FLOOR):
    """Explicit inverse of a 2x2 covariance; DegenerateCovariance below the det floor."""
    c = np.asarray(cov2, dtype=np.float64)
    det = c[0, 0] * c[1, 1] - c[0, 1] * c[1, 0]
    if det < det_floor:
        raise DegenerateCovariance(f"det {det} below floor {det_floor}")
    return np.array([[c[1, 1], -c[0, 1]], [-c[1, 0], c[0, 0]]]) / det


def _empty_map(view_id, w, h, degenerate):
    e = np.empty(0)
    return WeightMap(view_id, w, h, np.empty(0, np.int32), np.empty(0, np.int32),
                     np.empty(0, np.int64), e, e.copy(), e.copy(), degenerate)


def rasterize_weights(view, gaussians, alpha_cutoff=ALPHA_CUTOFF_DEFAULT,
                      early_stop=EARLY_STOP_TRANSMITTANCE, view_id=0) -> WeightMap:
    """GPU rasterizer with the reference's exact contribution set and order."""
    import torch

    from .core import gaussians_array
    from .engine import as_device

    if not 0.0 < alpha_cutoff < 1.0:
        raise ValueError(f"alpha_cutoff must be in (0, 1), got {alpha_cutoff}")
    w, h = int(view.width), int(view.height)
    rows = gaussians_array(gaussians)
    n = len(rows)
    if n == 0:
        return _empty_map(view_id, w, h, [])
    lib = nat.lib()
    plan = nat.default_plan()
    g = as_device(rows, torch.float64)
    cam = nat.make_camera(view)
    m = ctypes.c_int64(0)
    nd = ctypes.c_int64(0)
    stream = nat.stream_ptr()
    nat.check(lib.ts_rasterize_weights(plan.handle, nat.dptr(g), n, ctypes.byref(cam),
                                       float(alpha_cutoff), float(early_stop), ctypes.byref(m),
                                       ctypes.byref(nd), stream), "rasterize_weights")
    m, nd = int(m.value), int(nd.value)
    dev = g.device
    px = torch.empty(m, dtype=torch.int32, device=dev)
    py = torch.empty(m, dtype=torch.int32, device=dev)
    gid = torch.empty(m, dtype=torch.int64, device=dev)
    al = torch.empty(m, dtype=torch.float64, device=dev)
    tr = torch.empty(m, dtype=torch.float64, device=dev)
    de = torch.empty(m, dtype=torch.float64, device=dev)
    deg = torch.empty(max(nd, 1), dtype=torch.int64, device=dev)
    nat.check(lib.ts_rasterize_fetch(plan.handle, nat.dptr(px), nat.dptr(py), nat.dptr(gid),
                                     nat.dptr(al), nat.dptr(tr), nat.dptr(de), nat.dptr(deg),
                                     stream), "rasterize_fetch")
    degenerate = [int(i) for i in deg[:nd].cpu().numpy()]
    if m == 0:
        return _empty_map(view_id, w, h, degenerate)
    return WeightMap(view_id, w, h, px.cpu().numpy(), py.cpu().numpy(), gid.cpu().numpy(),
                     al.cpu().numpy(), tr.cpu().numpy(), de.cpu().numpy(), degenerate)
