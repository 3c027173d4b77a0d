"""ctypes binding of libtrackersplat_b200.so (include/trackersplat_b200.h).

The product path has no CPU fallback: importing the package works without a GPU (so host-side
types can be used and tested), but every hot-path call goes through `lib()`, which raises
`NativeUnavailable` if the CUDA library is missing or no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .errors import DimensionMismatch, GaussTrackError

_HERE = os.path.dirname(os.path.abspath(__file__))
# TS_LIB_PATH selects an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("TS_LIB_PATH") or os.path.join(_HERE, "_lib", "libtrackersplat_b200.so")
CSRC = os.path.join(_HERE, "csrc")

TS_OK = 0
TS_E_INVALID_ARGUMENT = -1
TS_E_DIMENSION_MISMATCH = -2
TS_E_CUDA = -3
TS_E_OUT_OF_MEMORY = -4
TS_E_CAPACITY = -5
TS_TRACK_F32 = 0
TS_TRACK_F64 = 1
N_STAGES = 6
STAGE_NAMES = ("k1_project", "depth_sort", "tile_sort", "k2_raster_accumulate", "k3_solve",
               "k4_fuse")


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing; there is deliberately no CPU fallback."""


class NativeError(GaussTrackError):
    """A CUDA-side failure reported through the C ABI."""


class Camera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("alpha_cutoff", ctypes.c_double), ("early_stop", ctypes.c_double),
                ("det_floor", ctypes.c_double), ("min_weight", ctypes.c_double),
                ("min_total_weight", ctypes.c_double), ("static_threshold_px", ctypes.c_double),
                ("eig_floor", ctypes.c_double), ("min_pixels", ctypes.c_int32),
                ("min_views", ctypes.c_int32), ("min_total_pixels", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_vp = ctypes.c_void_p


class Motions(ctypes.Structure):
    _fields_ = [("status", _vp), ("a", _vp), ("b", _vp), ("weight_sum", _vp),
                ("pixel_count", _vp), ("static_pixel_count", _vp), ("static_weight_sum", _vp)]


class Updates(ctypes.Structure):
    _fields_ = [("delta_mean", _vp), ("rotation", _vp), ("scale", _vp), ("status", _vp)]


class Binning(ctypes.Structure):
    _fields_ = [("n_instances", ctypes.c_int64), ("tiles_x", ctypes.c_int32),
                ("tiles_y", ctypes.c_int32), ("n_views", ctypes.c_int32), ("inst_tile", _vp),
                ("inst_gv", _vp), ("tile_range", _vp), ("gv_status", _vp), ("gv_bbox", _vp)]


class RegConfig(ctypes.Structure):
    _fields_ = [("min_hit_pixels", ctypes.c_int32), ("min_views", ctypes.c_int32),
                ("static_fraction", ctypes.c_double), ("average", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


TS_KNN_MAX_K = 32
_UP = ctypes.POINTER(Updates)

_SIGS = {
    "ts_version": ([], ctypes.c_int),
    "ts_error_string": ([ctypes.c_int], ctypes.c_char_p),
    "ts_plan_create": ([ctypes.POINTER(_vp)], ctypes.c_int),
    "ts_plan_destroy": ([_vp], ctypes.c_int),
    "ts_plan_workspace_bytes": ([_vp], ctypes.c_int64),
    "ts_plan_timing": ([_vp, ctypes.c_int], ctypes.c_int),
    "ts_plan_timing_read": ([_vp, _vp, _vp, ctypes.c_int32], ctypes.c_int),
    "ts_plan_set_k2_ctas_per_sm": ([_vp, ctypes.c_int32], ctypes.c_int),
    "ts_project": ([_vp, ctypes.c_int64, ctypes.POINTER(Camera), _vp, _vp, _vp, _vp, _vp],
                   ctypes.c_int),
    "ts_frame_bin": ([_vp, _vp, ctypes.c_int64, ctypes.POINTER(Camera), ctypes.c_int32,
                      ctypes.POINTER(Config), _vp], ctypes.c_int),
    "ts_frame_compensate": ([_vp, _vp, ctypes.c_int32, _vp, ctypes.POINTER(Motions),
                             ctypes.POINTER(Updates), _vp], ctypes.c_int),
    "ts_frame_binning": ([_vp, ctypes.POINTER(Binning)], ctypes.c_int),
    "ts_frame_occupied_tiles": ([_vp, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "ts_frame_track_rects": ([_vp, _vp], ctypes.c_int),
    "ts_frame_cache": ([_vp, ctypes.c_int32, _vp], ctypes.c_int),
    "ts_frame_cache_info": ([_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)],
                            ctypes.c_int),
    "ts_copy_track_rects": ([_vp, _vp, ctypes.c_int32, _vp, _vp, _vp, _vp], ctypes.c_int),
    "ts_rasterize_weights": ([_vp, _vp, ctypes.c_int64, ctypes.POINTER(Camera), ctypes.c_double,
                              ctypes.c_double, ctypes.POINTER(ctypes.c_int64),
                              ctypes.POINTER(ctypes.c_int64), _vp], ctypes.c_int),
    "ts_rasterize_fetch": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "ts_accumulate_view": ([_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int32,
                            ctypes.c_int32, _vp, ctypes.c_int32, _vp, ctypes.c_int64,
                            ctypes.c_double, _vp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "ts_solve_view": ([_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_double, ctypes.c_int32,
                       ctypes.c_double, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "ts_update_all": ([_vp, ctypes.c_int64, ctypes.POINTER(Camera), ctypes.c_int32,
                       ctypes.POINTER(Motions), ctypes.POINTER(Config), ctypes.POINTER(Updates),
                       _vp], ctypes.c_int),
    "ts_triangulate_batch": ([_vp, _vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp],
                             ctypes.c_int),
    "ts_solve_cov3d_batch": ([_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp],
                             ctypes.c_int),
    "ts_decompose_batch": ([_vp, _vp, ctypes.c_int64, ctypes.c_double, _vp, _vp, _vp, _vp],
                           ctypes.c_int),
    "ts_dominant_gaussians": ([_vp, ctypes.c_int32, _vp, _vp, _vp], ctypes.c_int),
    "ts_build_knn": ([_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _vp, _vp],
                     ctypes.c_int),
    "ts_detect_static": ([_vp, _vp, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(RegConfig),
                          _vp, _vp], ctypes.c_int),
    "ts_median_filter": ([_vp, ctypes.c_int64, _UP, _vp, ctypes.c_int32, _UP, _vp], ctypes.c_int),
    "ts_propagate": ([_vp, _vp, ctypes.c_int64, _UP, _vp, ctypes.c_int32, _vp, ctypes.c_int32,
                      _UP, _vp], ctypes.c_int),
    "ts_apply_updates": ([_vp, ctypes.c_int64, _UP, _vp, _vp], ctypes.c_int),
    "ts_regularize": ([_vp, _vp, ctypes.c_int64, _UP, _vp, _vp, ctypes.c_int32, _vp,
                       ctypes.c_int32, ctypes.POINTER(RegConfig), _UP, _vp, _vp, _vp],
                      ctypes.c_int),
    "ts_memcpy_d2h": ([_vp, _vp, ctypes.c_int64], ctypes.c_int),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_LIB = None


def build(verbose=False):
    """Compile the CUDA library for sm_100a with nvcc (in-tree, csrc/Makefile)."""
    out = subprocess.run(["make", "-s", "-C", CSRC, "-j8"], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("CUDA build failed:\n" + (out.stdout or "") + (out.stderr or ""))


def load_library(path=LIB_PATH):
    """dlopen the library and declare every C-ABI signature (no GPU needed)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(path):
            raise NativeUnavailable(f"{path} is not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = lib
    return _LIB


def lib():
    """The loaded library, after checking that a CUDA device is usable."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 hot path has no CPU fallback")
    return load_library()


def check(rc, what="call"):
    if rc == TS_OK:
        return
    msg = f"{what} failed: {load_library().ts_error_string(rc).decode()} ({rc})"
    if rc == TS_E_DIMENSION_MISMATCH:
        raise DimensionMismatch(msg)
    if rc == TS_E_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise NativeError(msg)


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def make_camera(cam) -> Camera:
    """ts_camera from a CameraView-like object or an 18-vector (R9, t3, fx, fy, cx, cy, W, H)."""
    c = Camera()
    if hasattr(cam, "rotation"):
        r = np.asarray(cam.rotation, np.float64).ravel()
        t = np.asarray(cam.translation, np.float64).ravel()
        vals = (cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    else:
        a = np.asarray(cam, np.float64).ravel()
        r, t, vals = a[:9], a[9:12], a[12:18]
    for i in range(9):
        c.R[i] = float(r[i])
    for i in range(3):
        c.t[i] = float(t[i])
    c.fx, c.fy, c.cx, c.cy = (float(v) for v in vals[:4])
    c.width, c.height = int(vals[4]), int(vals[5])
    return c


def make_cameras(cams):
    arr = (Camera * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = make_camera(c)
    return arr


def make_reg_config(cfg=None, average=None) -> RegConfig:
    """ts_reg_config from a Config (pipeline.py:88-96 fields)."""
    c = RegConfig()
    get = (lambda k, d: getattr(cfg, k, d)) if cfg is not None else (lambda k, d: d)
    c.min_hit_pixels = int(get("min_hit_pixels", 9))
    c.min_views = int(get("min_views", 2))
    c.static_fraction = float(get("static_fraction", 0.9))
    avg = average if average is not None else get("propagation_average", "mean")
    if avg not in ("mean", "median"):
        raise ValueError(f"average must be 'mean' or 'median', got {avg}")
    c.average = 0 if avg == "mean" else 1
    return c


def make_config(cfg=None, early_stop=1e-4) -> Config:
    c = Config()
    get = (lambda k, d: getattr(cfg, k, d)) if cfg is not None else (lambda k, d: d)
    c.alpha_cutoff = float(get("alpha_cutoff", 1.0 / 255.0))
    c.early_stop = float(early_stop)
    c.det_floor = float(get("det_floor", 1e-12))
    c.min_weight = float(get("min_weight", 1e-3))
    c.min_total_weight = float(get("min_total_weight", 1e-3))
    c.static_threshold_px = float(get("static_threshold_px", 1.0))
    c.eig_floor = float(get("eig_floor", 1e-12))
    c.min_pixels = int(get("min_pixels", 3))
    c.min_views = int(get("min_views", 2))
    c.min_total_pixels = int(get("min_total_pixels", 3))
    c.reserved = 0
    return c


class Plan:
    """Owns a ts_plan (grow-only device workspace); one per device/stream user."""

    def __init__(self):
        self._lib = lib()
        h = ctypes.c_void_p()
        check(self._lib.ts_plan_create(ctypes.byref(h)), "ts_plan_create")
        self.handle = h
        self.k2_ctas_per_sm = 0

    def close(self):
        if self.handle:
            self._lib.ts_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def workspace_bytes(self):
        return int(self._lib.ts_plan_workspace_bytes(self.handle))

    def timing(self, enable=True):
        check(self._lib.ts_plan_timing(self.handle, int(bool(enable))), "ts_plan_timing")

    def set_k2_ctas_per_sm(self, ctas_per_sm):
        """Cap the persistent K2 grid at `ctas_per_sm` CTAs per SM (0: full residency)."""
        check(self._lib.ts_plan_set_k2_ctas_per_sm(self.handle, int(ctas_per_sm)),
              "ts_plan_set_k2_ctas_per_sm")
        self.k2_ctas_per_sm = int(ctas_per_sm)

    def timing_read(self):
        tot = (ctypes.c_double * N_STAGES)()
        cnt = (ctypes.c_int32 * N_STAGES)()
        check(self._lib.ts_plan_timing_read(self.handle, ctypes.cast(tot, _vp),
                                            ctypes.cast(cnt, _vp), N_STAGES), "timing_read")
        return {STAGE_NAMES[i]: (tot[i], cnt[i]) for i in range(N_STAGES)}


_DEFAULT_PLAN = {}


def default_plan():
    """A per-device Plan shared by the stage-API shims."""
    import torch
    dev = torch.cuda.current_device()
    p = _DEFAULT_PLAN.get(dev)
    if p is None:
        p = _DEFAULT_PLAN[dev] = Plan()
    return p
