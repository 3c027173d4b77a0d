"""Batched, tensor-native engine of the hot path (the fused K1 -> K2 -> K3 -> K4 pipeline).

This is the fast path under `compensate_frame`: Gaussians, cameras and tracks stay on the device
as SoA tensors; reference-typed objects are only produced on demand by the API shims.

    eng = FrameEngine()
    eng.bin(gaussians, cameras, config)          # K1: once per clip (pipeline.py:191-196)
    out = eng.compensate(track_target, valid)    # K2 + K3 + K4: once per target frame

Layouts (device):
    gaussians     (N, 11) float64    mean, quaternion (w,x,y,z), scale, opacity
    track_target  (V, H, W, 2)       float32 (TRKF, fileio.py:108-136) or float64
    track_valid   (V, H, W)          uint8
    motions       SoA over gv = v*N + g: status int8, a (.,2,2) f64, b (.,2) f64,
                  weight_sum f64, pixel_count i32, static_pixel_count i32, static_weight_sum f64
    updates       delta_mean (N,3), rotation (N,4), scale (N,3) f64, status int8
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import cameras_array, gaussians_array


def _nullctx():
    import contextlib
    return contextlib.nullcontext()


def _torch():
    import torch
    return torch


def _pinned(t):
    """True for a contiguous page-locked CPU tensor, which kernels may read in place."""
    torch = _torch()
    return (isinstance(t, torch.Tensor) and t.device.type == "cpu" and t.is_contiguous()
            and t.is_pinned())


def _pinned_pair(tgt, val):
    return _pinned(tgt) and _pinned(val)


def as_device(x, dtype, device=None):
    """Host array / tensor -> contiguous CUDA tensor of `dtype` (no copy if already there)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    if t.device != dev or t.dtype != dtype:
        t = t.to(device=dev, dtype=dtype, non_blocking=False)
    return t.contiguous()


@dataclass
class FrameOutputs:
    delta_mean: "object"
    rotation: "object"
    scale: "object"
    status: "object"
    motion_status: "object"
    motion_a: "object"
    motion_b: "object"
    weight_sum: "object"
    pixel_count: "object"
    static_pixel_count: "object"
    static_weight_sum: "object"

    def tallies(self):
        st = self.status
        return {"solved": int((st == 1).sum()), "static": int((st == 2).sum()),
                "unsolvable": int((st == 0).sum())}


MAX_VIEWS_PER_PLAN = 64  # view bits of K1's 32-bit depth key (api.cu frame_bin)


def view_groups(cam_rows, max_views=MAX_VIEWS_PER_PLAN):
    """Consecutive runs of views with the same image size, at most `max_views` each: the unit one
    binning plan handles (K1-K3); K4 then fuses every view at once."""
    groups, v0 = [], 0
    for v in range(1, len(cam_rows) + 1):
        if (v == len(cam_rows) or v - v0 == max_views or
                tuple(cam_rows[v][16:18]) != tuple(cam_rows[v0][16:18])):
            groups.append((v0, v))
            v0 = v
    return groups


class FrameEngine:
    """Holds the per-clip binning and per-frame workspace of one device.

    The reference rasterizes every view at its own size (pipeline.py:117-120) and accepts any
    number of views.  One binning plan covers up to 64 views of one image size; other camera
    rigs are binned as consecutive same-size groups of <= 64 views, each with its own plan for
    K1-K3, and K4 fuses all views at once (ts_update_all).  Tracks of such rigs are passed as
    per-view lists."""

    def __init__(self, plan: nat.Plan | None = None):
        self.plan = plan if plan is not None else nat.Plan()
        self._lib = nat.lib()
        self.n = 0
        self.n_views = 0
        self.width = self.height = 0
        self._gauss = None
        self._cams = None
        self._groups = None  # [(v0, v1, Plan)] when the views need more than one plan
        self._sizes = []

    @property
    def grouped(self):
        return self._groups is not None

    # -- K1 ------------------------------------------------------------------------------
    def bin(self, gaussians, cameras, config=None, stream=None):
        """Project + depth-order + tile-bin the first-frame Gaussians into every view."""
        torch = _torch()
        g = gaussians if isinstance(gaussians, torch.Tensor) else gaussians_array(gaussians)
        self._gauss = as_device(g, torch.float64).reshape(-1, 11)
        cam_rows = cameras_array(cameras)
        self._cams = nat.make_cameras(cam_rows)
        self._cfg = nat.make_config(config)
        self.n = int(self._gauss.shape[0])
        self.n_views = len(cam_rows)
        self.width, self.height = int(cam_rows[0][16]), int(cam_rows[0][17])
        self._sizes = [(int(r[16]), int(r[17])) for r in cam_rows]
        groups = view_groups(cam_rows)
        if len(groups) == 1:
            self._groups = None
            nat.check(self._lib.ts_frame_bin(self.plan.handle, nat.dptr(self._gauss), self.n,
                                             self._cams, self.n_views, ctypes.byref(self._cfg),
                                             nat.stream_ptr(stream)), "ts_frame_bin")
            return self
        old = {(v0, v1): p for v0, v1, p in (self._groups or [])}
        self._groups = []
        for k, (v0, v1) in enumerate(groups):
            plan = self.plan if k == 0 else old.get((v0, v1)) or nat.Plan()
            sub = nat.make_cameras(cam_rows[v0:v1])
            nat.check(self._lib.ts_frame_bin(plan.handle, nat.dptr(self._gauss), self.n, sub,
                                             v1 - v0, ctypes.byref(self._cfg),
                                             nat.stream_ptr(stream)), "ts_frame_bin")
            self._groups.append((v0, v1, plan))
        return self

    def _group_of(self, view):
        for v0, v1, plan in self._groups:
            if v0 <= view < v1:
                return v0, plan
        raise IndexError(view)

    def binning(self):
        """Copies of the binning arrays (tile keys, instance order, ranges, bbox, status)."""
        torch = _torch()
        if self.grouped:
            raise NotImplementedError("binning() of a grouped (multi-plan) camera rig")
        b = nat.Binning()
        nat.check(self._lib.ts_frame_binning(self.plan.handle, ctypes.byref(b)), "binning")
        torch.cuda.synchronize()
        ni = int(b.n_instances)
        nt = int(b.tiles_x) * int(b.tiles_y) * int(b.n_views)
        nv = self.n * self.n_views

        def grab(ptr, count, dtype, width=1):
            out = np.empty(count * width, dtype)
            if count:
                nat.check(self._lib.ts_memcpy_d2h(out.ctypes.data, ptr, out.nbytes), "d2h")
            return out.reshape(count, width) if width > 1 else out

        return dict(n_instances=ni, tiles_x=int(b.tiles_x), tiles_y=int(b.tiles_y),
                    inst_tile=grab(b.inst_tile, ni, np.uint32),
                    inst_gv=grab(b.inst_gv, ni, np.uint32),
                    tile_range=grab(b.tile_range, nt, np.uint32, 2),
                    status=grab(b.gv_status, nv, np.int8),
                    bbox=grab(b.gv_bbox, nv, np.int16, 4))

    def build_cache(self, stream=None):
        """Rasterize the current binning once WITHOUT tracks and keep every contribution (pixel,
        w = alpha T) for the clip: later compensate() calls apply each target frame's tracks to
        the cache instead of re-rasterizing (the reference reuses the frame-0 weight maps across
        a clip's target frames, pipeline.py:191-196).  Valid until the next bin()."""
        plans = [self.plan] if not self.grouped else [g[2] for g in self._groups]
        for plan in plans:
            nat.check(self._lib.ts_frame_cache(plan.handle, 1, nat.stream_ptr(stream)),
                      "ts_frame_cache")
        return self

    def cache_info(self):
        """(records, cached w values) of the current clip cache, summed over the plans."""
        import ctypes
        plans = [self.plan] if not self.grouped else [g[2] for g in self._groups]
        tot = [0, 0]
        for plan in plans:
            r, v = ctypes.c_uint64(), ctypes.c_uint64()
            nat.check(self._lib.ts_frame_cache_info(plan.handle, ctypes.byref(r), ctypes.byref(v)),
                      "ts_frame_cache_info")
            tot[0] += r.value
            tot[1] += v.value
        return tuple(tot)

    def drop_cache(self):
        plans = [self.plan] if not self.grouped else [g[2] for g in self._groups]
        for plan in plans:
            nat.check(self._lib.ts_frame_cache(plan.handle, 0, None), "ts_frame_cache")
        return self

    def track_rects(self):
        """(V, 4) int32 inclusive pixel rectangles (x0, y0, x1, y1) the next compensate reads."""
        if self.grouped:
            raise NotImplementedError("track_rects() of a grouped (multi-plan) camera rig")
        r = np.empty((self.n_views, 4), np.int32)
        nat.check(self._lib.ts_frame_track_rects(self.plan.handle, r.ctypes.data), "track_rects")
        return r

    def copy_track_rects(self, t_host, v_host, t_dev, v_dev, stream=None):
        """DMA the track rectangles of the current binning from pinned host tensors into device
        tensors of the same layout, on `stream` (asynchronous)."""
        torch = _torch()
        if self.grouped:  # several plans: the whole arrays (the rig is binned per view group)
            with torch.cuda.stream(stream) if stream is not None else _nullctx():
                t_dev.copy_(t_host, non_blocking=True)
                v_dev.copy_(v_host, non_blocking=True)
            return
        dtype = nat.TS_TRACK_F32 if t_host.dtype == torch.float32 else nat.TS_TRACK_F64
        nat.check(self._lib.ts_copy_track_rects(self.plan.handle, t_host.data_ptr(), dtype,
                                                v_host.data_ptr(), t_dev.data_ptr(),
                                                v_dev.data_ptr(), nat.stream_ptr(stream)),
                  "copy_track_rects")

    def occupied_tiles(self):
        """Non-empty (view, tile) lists of the current binning (K2 reads 256 track pixels each)."""
        total = 0
        for plan in ([self.plan] if not self.grouped else [g[2] for g in self._groups]):
            c = ctypes.c_int64(0)
            nat.check(self._lib.ts_frame_occupied_tiles(plan.handle, ctypes.byref(c)),
                      "occupied_tiles")
            total += int(c.value)
        return total

    # -- K2 + K3 + K4 ----------------------------------------------------------------------
    MOTION_FIELDS = ("motion_status", "motion_a", "motion_b", "weight_sum", "pixel_count",
                     "static_pixel_count", "static_weight_sum")

    def alloc_outputs(self, motions=True):
        """Output buffers of compensate().  motions=False: the updates only -- the per-view
        motions are intermediates of compensate_frame (pipeline.py:117-124; FrameResult carries
        the updated Gaussians), so K3 may keep its fits compact and K4 read them in place."""
        torch = _torch()
        n, nv = self.n, self.n * self.n_views
        dev = self._gauss.device
        f64 = dict(dtype=torch.float64, device=dev)
        if not motions:
            return FrameOutputs(
                delta_mean=torch.empty((n, 3), **f64), rotation=torch.empty((n, 4), **f64),
                scale=torch.empty((n, 3), **f64),
                status=torch.empty(n, dtype=torch.int8, device=dev),
                **{k: None for k in self.MOTION_FIELDS})
        return FrameOutputs(
            delta_mean=torch.empty((n, 3), **f64), rotation=torch.empty((n, 4), **f64),
            scale=torch.empty((n, 3), **f64), status=torch.empty(n, dtype=torch.int8, device=dev),
            motion_status=torch.empty(nv, dtype=torch.int8, device=dev),
            motion_a=torch.empty((nv, 2, 2), **f64), motion_b=torch.empty((nv, 2), **f64),
            weight_sum=torch.empty(nv, **f64),
            pixel_count=torch.empty(nv, dtype=torch.int32, device=dev),
            static_pixel_count=torch.empty(nv, dtype=torch.int32, device=dev),
            static_weight_sum=torch.empty(nv, **f64))

    def outputs_fit(self, out: FrameOutputs) -> bool:
        """True if `out` has this engine's shapes (N Gaussians, N x V fits) on its device."""
        n, nv = self.n, self.n * self.n_views
        dev = self._gauss.device
        want = dict(delta_mean=(n, 3), rotation=(n, 4), scale=(n, 3), status=(n,),
                    motion_status=(nv,), motion_a=(nv, 2, 2), motion_b=(nv, 2),
                    weight_sum=(nv,), pixel_count=(nv,), static_pixel_count=(nv,),
                    static_weight_sum=(nv,))
        no_motions = all(getattr(out, k) is None for k in self.MOTION_FIELDS)
        for k, shape in want.items():
            t = getattr(out, k)
            if t is None and no_motions and k in self.MOTION_FIELDS:
                continue
            if t is None or tuple(t.shape) != shape or t.device != dev or not t.is_contiguous():
                return False
        return True

    def check_outputs(self, out: FrameOutputs):
        """Reject a caller's output buffers that the kernels would overrun."""
        if not self.outputs_fit(out):
            raise ValueError(f"output buffers do not match this engine's binning "
                             f"(N={self.n}, views={self.n_views}); use alloc_outputs()")

    def compensate(self, track_target, track_valid, out: FrameOutputs | None = None,
                   stream=None, motions=True) -> FrameOutputs:
        """Fused raster-accumulate, per-view affine fit and multi-view fuse for one frame.

        Tracks: (V, H, W, 2) targets and (V, H, W) validity (device tensors, pinned host tensors
        read in place by K2, or host arrays that are copied), or per-view lists of them (required
        when the views differ in size)."""
        torch = _torch()
        if self._gauss is None:
            raise RuntimeError("FrameEngine.bin() must run before compensate()")
        if self.grouped or isinstance(track_target, (list, tuple)):
            return self._compensate_groups(track_target, track_valid, out, stream, motions)
        tgt, val = track_target, track_valid
        # each array: a CUDA tensor as is; a pinned CPU tensor is read in place by K2 (zero-copy:
        # only the occupied tiles' quadrants cross PCIe); anything else is copied to the device
        if _pinned(tgt):
            if tgt.dtype not in (torch.float32, torch.float64):
                raise TypeError("pinned track targets must be float32 or float64")
        elif not isinstance(tgt, torch.Tensor):
            tgt = np.asarray(tgt)
            tgt = as_device(tgt, torch.float32 if tgt.dtype == np.float32 else torch.float64)
        else:
            tgt = tgt.contiguous()
            if tgt.device.type != "cuda":
                tgt = as_device(tgt, tgt.dtype)
        if _pinned(val):
            if val.dtype != torch.uint8:
                raise TypeError("pinned track validity must be uint8")
        else:
            val = as_device(val, torch.uint8)
        expect = (self.n_views, self.height, self.width)
        if tuple(tgt.shape) != expect + (2,) or tuple(val.shape) != expect:
            from .errors import DimensionMismatch
            raise DimensionMismatch(f"tracks {tuple(tgt.shape)} / {tuple(val.shape)} do not "
                                    f"match {expect}")
        dtype = nat.TS_TRACK_F32 if tgt.dtype == torch.float32 else nat.TS_TRACK_F64
        if out is None:
            out = self.alloc_outputs(motions)
        else:
            self.check_outputs(out)
        m = None
        if out.motion_status is not None:
            m = ctypes.byref(nat.Motions(
                nat.dptr(out.motion_status).value, nat.dptr(out.motion_a).value,
                nat.dptr(out.motion_b).value, nat.dptr(out.weight_sum).value,
                nat.dptr(out.pixel_count).value, nat.dptr(out.static_pixel_count).value,
                nat.dptr(out.static_weight_sum).value))
        u = nat.Updates(nat.dptr(out.delta_mean).value, nat.dptr(out.rotation).value,
                        nat.dptr(out.scale).value, nat.dptr(out.status).value)
        nat.check(self._lib.ts_frame_compensate(self.plan.handle, nat.dptr(tgt), dtype,
                                                nat.dptr(val), m, ctypes.byref(u),
                                                nat.stream_ptr(stream)), "ts_frame_compensate")
        return out

    def _track_pair(self, tgt, val):
        """One (..., 2) target / validity pair as the C ABI takes it: device or pinned host."""
        torch = _torch()
        if _pinned(tgt):
            if tgt.dtype not in (torch.float32, torch.float64):
                raise TypeError("pinned track targets must be float32 or float64")
        elif not isinstance(tgt, torch.Tensor):
            tgt = np.asarray(tgt)
            tgt = as_device(tgt, torch.float32 if tgt.dtype == np.float32 else torch.float64)
        else:
            tgt = tgt.contiguous()
            if tgt.device.type != "cuda":
                tgt = as_device(tgt, tgt.dtype)
        if _pinned(val):
            if val.dtype != torch.uint8:
                raise TypeError("pinned track validity must be uint8")
        else:
            val = as_device(val, torch.uint8)
        return tgt, val

    def _compensate_groups(self, targets, valids, out, stream, motions=True):
        """Per-view track lists, and rigs binned as several plans: K2+K3 per plan into the
        plan's slice of the view-major motion arrays, then K4 over every view."""
        torch = _torch()
        from .errors import DimensionMismatch
        if len(targets) != self.n_views or len(valids) != self.n_views:
            raise DimensionMismatch("track fields and cameras count differ")
        tv = []
        for v in range(self.n_views):
            tgt, val = self._track_pair(targets[v], valids[v])
            w, h = self._sizes[v]
            if tuple(tgt.shape) != (h, w, 2) or tuple(val.shape) != (h, w):
                raise DimensionMismatch(f"view {v}: tracks {tuple(tgt.shape)} / "
                                        f"{tuple(val.shape)} vs camera {w}x{h}")
            tv.append((tgt, val))
        if out is None:
            out = self.alloc_outputs(motions)
        else:
            self.check_outputs(out)
        if out.motion_status is None:  # the fuse over all views reads the dense motions
            full = self.alloc_outputs()
            for k in ("delta_mean", "rotation", "scale", "status"):
                setattr(full, k, getattr(out, k))
            out = full
        groups = self._groups or [(0, self.n_views, self.plan)]
        n = self.n
        for v0, v1, plan in groups:
            dt = torch.float64 if any(t.dtype == torch.float64 for t, _ in tv[v0:v1]) \
                else torch.float32
            tgt = torch.stack([t.to("cuda", dt) for t, _ in tv[v0:v1]])
            val = torch.stack([x.to("cuda") for _, x in tv[v0:v1]])
            off = v0 * n

            def at(t, k=1):
                return nat.dptr(t).value + off * k * t.element_size()
            m = nat.Motions(at(out.motion_status), at(out.motion_a, 4), at(out.motion_b, 2),
                            at(out.weight_sum), at(out.pixel_count), at(out.static_pixel_count),
                            at(out.static_weight_sum))
            nat.check(self._lib.ts_frame_compensate(
                plan.handle, nat.dptr(tgt),
                nat.TS_TRACK_F32 if dt == torch.float32 else nat.TS_TRACK_F64, nat.dptr(val),
                ctypes.byref(m), None, nat.stream_ptr(stream)), "ts_frame_compensate")
        m = nat.Motions(nat.dptr(out.motion_status).value, nat.dptr(out.motion_a).value,
                        nat.dptr(out.motion_b).value, nat.dptr(out.weight_sum).value,
                        nat.dptr(out.pixel_count).value, nat.dptr(out.static_pixel_count).value,
                        nat.dptr(out.static_weight_sum).value)
        u = nat.Updates(nat.dptr(out.delta_mean).value, nat.dptr(out.rotation).value,
                        nat.dptr(out.scale).value, nat.dptr(out.status).value)
        nat.check(self._lib.ts_update_all(nat.dptr(self._gauss), n, self._cams, self.n_views,
                                          ctypes.byref(m), ctypes.byref(self._cfg),
                                          ctypes.byref(u), nat.stream_ptr(stream)),
                  "ts_update_all")
        return out

    def dominant_gaussians(self, view, stream=None):
        """Per-pixel dominant Gaussian id (-1 if none) and its depth (scene.py:166-189)."""
        torch = _torch()
        w, h = self._sizes[view]
        gid = torch.empty((h, w), dtype=torch.int64, device="cuda")
        dep = torch.empty((h, w), dtype=torch.float64, device="cuda")
        v0, plan = self._group_of(view) if self.grouped else (0, self.plan)
        nat.check(self._lib.ts_dominant_gaussians(plan.handle, int(view - v0), nat.dptr(gid),
                                                  nat.dptr(dep), nat.stream_ptr(stream)),
                  "ts_dominant_gaussians")
        return gid, dep


class StreamingEngine:
    """Pipelined end-to-end driver: pinned host inputs in, pinned host results out.

    Streams: one H2D stream, N_ENGINES compute streams and one D2H stream.  `step(inputs_k)` enqueues
    the H2D copy of step k's inputs and then the compute of the PREVIOUS step (k-1), so the copy
    of step k is already queued when step k-1's binning briefly synchronises the host (the
    instance count).  Consecutive steps compute on alternating engines (binning plans) and
    compute streams, so N_ENGINES frames are in flight: one frame's binning fills the SMs that the
    other's latency-bound K3/K4 leave idle.  The D2H of a step's results runs on its own stream
    from that engine's output buffer.  Tracks given as pinned host tensors need not be copied
    (`zero_copy_tracks=True`): K2 reads the 8x8 quadrants of the occupied tiles in place over
    PCIe (about a tenth of the track bytes at the benchmark configs, but at the PCIe request rate
    rather than its bandwidth); with `zero_copy_tracks=False` the whole arrays are copied on the
    H2D stream (DMA at full bandwidth, hidden when the compute takes longer).  The default
    `"rect"` copies, once the frame's binning is known, only the pixel rectangles of the tiles
    K2 will read (ts_copy_track_rects: a third of the track bytes at cfg2) with the copy engine
    while the other frames in flight compute -- never slower than the best of the other two by
    more than ~1% on the BASELINE configs, faster at cfg2 / cfg5.  `"auto"` picks per step
    between reading in place and the whole copy from measured step periods.  All modes give
    bit-identical results.  Input slots and
    output buffers are reused in turn, ordered with CUDA events.  `step` returns the event after
    which the previous step's results are in its host buffer (None for the first call);
    `flush()` runs the last pending step; `wait_all(stream)` orders `stream` after every result
    copy issued so far.  The caller must leave step k's host inputs unchanged until the event
    returned by the call that computes step k has completed.
    """

    N_ENGINES = 3  # frames in flight (cfg2 e2e, in place: 2 -> 4.15 ms, 3 -> 3.92 ms per step)
    N_SLOTS = N_ENGINES + 2  # input slots: the copy of step k+1 never waits for a frame in flight
    H2D_GBS = 50.0  # pinned host -> device DMA rate assumed by the "auto" mode (GB/s)
    # K2 residency of the engines (ts_plan_set_k2_ctas_per_sm): with frames in flight the
    # persistent K2 grid capped at 3 CTAs per SM leaves room for the other frame's kernels
    # (cfg2 e2e 4.45 -> 4.15 ms; K2 alone is slower, 2.10 -> 3.06 ms, so a frame run alone keeps
    # the full grid)
    K2_CTAS_PER_SM = 3

    SWITCH_VOTES = 3  # consecutive steps that must favour the other mode before "auto" switches
    SETTLE_STEPS = N_ENGINES + 2  # first steps (allocation, plan growth) never feed a period

    def __init__(self, engine: FrameEngine | None = None, zero_copy_tracks="rect"):
        torch = _torch()
        self._compute_ms = None  # median of the last in-place step periods ("auto" mode)
        self._periods = []
        self._copy_ms_meas = None  # median of the last full-copy step periods
        self._copy_periods = []
        self._n_timed = 0
        self._last_zero_copy = True
        self._votes = 0
        self._burst = 0
        self.steps_zero_copy = 0  # steps whose tracks were read in place / copied whole /
        self.steps_full_copy = 0  # copied as the tiles the frame reads ("rect")
        self.steps_rect_copy = 0
        self._rect_bytes = None  # track bytes of the last frame's rectangles ("rect" mode)
        self._timing = []  # (start, end) events of computed steps not yet read
        self.engines = [engine if engine is not None else FrameEngine()] + \
            [FrameEngine() for _ in range(self.N_ENGINES - 1)]
        # the K2 cap applies while this streamer runs; close() restores a passed-in engine's
        self._caller_cap = engine.plan.k2_ctas_per_sm if engine is not None else None
        for e_ in self.engines:
            e_.plan.set_k2_ctas_per_sm(self.K2_CTAS_PER_SM)
        self.zero_copy_tracks = zero_copy_tracks
        self.copy_stream = torch.cuda.Stream()
        self.rect_stream = torch.cuda.Stream()
        self.comp_streams = [torch.cuda.Stream() for _ in range(self.N_ENGINES)]
        self.d2h_stream = torch.cuda.Stream()
        self._slots = [None] * self.N_SLOTS
        self._free = [None] * self.N_SLOTS  # input slot i reusable after this compute event
        self._outs = [None] * self.N_ENGINES
        self._out_free = [None] * self.N_ENGINES  # engine e's outputs reusable after this D2H
        self._k = 0
        self._c = 0
        self._pending = None

    @property
    def eng(self):
        return self.engines[0]

    @property
    def comp_stream(self):
        return self.comp_streams[0]

    def _slot(self, i, g_host, t_host, v_host, tracks):
        torch = _torch()
        s = self._slots[i]
        shapes = (tuple(g_host.shape), tuple(t_host.shape), tuple(v_host.shape), t_host.dtype,
                  tracks)
        if s is None or s[0] != shapes:
            if s is not None and self._free[i] is not None:
                # the old buffers go back to the caching allocator: no stream may still use them
                self._free[i].synchronize()
            dev = torch.device("cuda", torch.cuda.current_device())
            s = (shapes, torch.empty(g_host.shape, dtype=torch.float64, device=dev),
                 torch.empty(t_host.shape, dtype=t_host.dtype, device=dev) if tracks else None,
                 torch.empty(v_host.shape, dtype=torch.uint8, device=dev) if tracks else None)
            self._slots[i] = s
        return s[1], s[2], s[3]

    @staticmethod
    def result_buffer(n):
        """Pinned host buffer for one step's result rows: delta(3) rotation(4) scale(3) status."""
        torch = _torch()
        return torch.empty((n, 11), dtype=torch.float64).pin_memory()

    def _compute(self, pending):
        torch = _torch()
        i, g_d, t_d, v_d, ready, cameras, res_host, config, src = pending
        e = self._c % self.N_ENGINES
        self._c += 1
        eng, cs = self.engines[e], self.comp_streams[e]
        cs.wait_event(ready)
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(cs)
        eng.bin(g_d, cameras, config, stream=cs)
        if src is not None:
            # "rect": the binning is known, so only the tiles K2 will read are DMA'd (the copy
            # engine works while the SMs run the other frames in flight).  A stream of its own:
            # on the input stream the copy would queue behind the next step's Gaussian copy,
            # which nothing waits for yet; `ready` (this slot's Gaussians) already ordered it
            # after the slot's previous use.
            self.rect_stream.wait_event(ready)
            eng.copy_track_rects(src[0], src[1], t_d, v_d, self.rect_stream)
            if not eng.grouped:
                r = eng.track_rects().astype(np.int64)
                px = int(np.sum(np.maximum(r[:, 2] - r[:, 0] + 1, 0) *
                                np.maximum(r[:, 3] - r[:, 1] + 1, 0)))
                self._rect_bytes = px * (2 * src[0].element_size() + 1)
            copied = torch.cuda.Event()
            copied.record(self.rect_stream)
            cs.wait_event(copied)
        # the binning does not touch the outputs: only K2-K4 wait for their previous D2H
        if self._out_free[e] is not None:
            cs.wait_event(self._out_free[e])
        if self._outs[e] is not None and not eng.outputs_fit(self._outs[e]):
            if self._out_free[e] is not None:
                self._out_free[e].synchronize()  # shapes changed: reallocate after the last D2H
            self._outs[e] = None
        # the host result is the updated Gaussians: no per-view motions (K4 reads K3's fits)
        out = eng.compensate(t_d, v_d, self._outs[e], stream=cs, motions=False)
        self._outs[e] = out
        computed = torch.cuda.Event(enable_timing=True)
        computed.record(cs)
        if self.zero_copy_tracks == "auto":
            self._n_timed += 1
            settled = self._n_timed > self.SETTLE_STEPS
            self._timing.append((t0, computed, self._burst if settled else -self._n_timed,
                                 t_d is not None and _pinned(t_d)))
        self._free[i] = computed
        ds = self.d2h_stream
        ds.wait_event(computed)
        with torch.cuda.stream(ds):
            # rows packed on the D2H stream, not the compute stream: a kernel queued there after K4
            # waits for the other frame's persistent K2 and holds back the next frame's binning
            res = torch.cat([out.delta_mean, out.rotation, out.scale,
                             out.status.to(torch.float64)[:, None]], 1)
            res_host.copy_(res, non_blocking=True)
            done = torch.cuda.Event()
            done.record(ds)
        self._out_free[e] = done
        self.out = out
        return done

    def step(self, g_host, cameras, t_host, v_host, res_host, config=None):
        """Enqueue the H2D copy of this step's inputs, then compute the previous step."""
        torch = _torch()
        i = self._k % self.N_SLOTS
        self._k += 1
        rect = self.zero_copy_tracks == "rect" and _pinned_pair(t_host, v_host)
        if rect and self._rect_bytes is not None:
            # whole arrays at most twice the last frame's rectangles: copy them before the
            # binning instead (off the frame's critical path; cfg3: 56 MB vs 29 MB of rectangles)
            whole = t_host.numel() * t_host.element_size() + v_host.numel()
            rect = whole > 2 * self._rect_bytes
        if self.zero_copy_tracks == "rect":
            zero_copy = False  # rectangles after the binning, or the whole arrays now
        else:
            zero_copy = self._choose_zero_copy(g_host, t_host, v_host) and \
                _pinned_pair(t_host, v_host)
        if rect:
            self.steps_rect_copy += 1
        elif zero_copy:
            self.steps_zero_copy += 1
        else:
            self.steps_full_copy += 1
        # "auto" keeps device track buffers in every slot, so a mode switch never allocates
        g_d, t_d, v_d = self._slot(i, g_host, t_host, v_host,
                                   not zero_copy or self.zero_copy_tracks == "auto")
        with torch.cuda.stream(self.copy_stream):
            if self._free[i] is not None:
                self.copy_stream.wait_event(self._free[i])
            g_d.copy_(g_host, non_blocking=True)
            if zero_copy:
                t_d, v_d = t_host, v_host  # read in place by K2
            elif not rect:
                t_d.copy_(t_host, non_blocking=True)
                v_d.copy_(v_host, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(self.copy_stream)
        src = (t_host, v_host) if rect else None  # rectangles copied after the binning
        prev, self._pending = self._pending, (i, g_d, t_d, v_d, ready, cameras, res_host, config,
                                              src)
        return self._compute(prev) if prev is not None else None

    def _choose_zero_copy(self, g_host, t_host, v_host):
        if self.zero_copy_tracks != "auto":
            return bool(self.zero_copy_tracks)
        # Fold in the step periods (interval between consecutive finished steps; never blocks),
        # one estimate per track mode from windows whose steps all used that mode.  Steps finish
        # on N_ENGINES compute streams, so a period is read once every event of the window has
        # completed; windows across a flush (caller's idle time) or within the first
        # SETTLE_STEPS steps (allocations) are skipped.
        k = self.N_ENGINES
        while len(self._timing) > k and all(t[1].query() for t in self._timing[:k + 1]):
            window = self._timing[:k + 1]
            first, last = window[0], window[-1]
            self._timing.pop(0)
            if first[2] != last[2] or first[2] < 0:
                continue
            period = first[1].elapsed_time(last[1]) / k
            if all(t[3] for t in window):
                self._periods = (self._periods + [period])[-5:]
                self._compute_ms = sorted(self._periods)[len(self._periods) // 2]
            elif not any(t[3] for t in window):
                self._copy_periods = (self._copy_periods + [period])[-5:]
                self._copy_ms_meas = sorted(self._copy_periods)[len(self._copy_periods) // 2]
        if self._compute_ms is None:
            return self._last_zero_copy
        copy_ms = (g_host.numel() * g_host.element_size() + t_host.numel() *
                   t_host.element_size() + v_host.numel()) / (self.H2D_GBS * 1e6)
        if self._last_zero_copy:
            # reading in place: copy the whole arrays when copying steps were measured faster,
            # or (never measured) when the estimated copy hides under the period
            if self._copy_ms_meas is not None:
                want_zero_copy = not self._copy_ms_meas < 0.97 * self._compute_ms
            else:
                want_zero_copy = not copy_ms < 0.85 * self._compute_ms
        else:
            # copying: go back once the copying steps are measured slower than in-place ones
            # (the copy sits in their period, so the in-place estimate is never refreshed here)
            want_zero_copy = (self._copy_ms_meas is not None and
                              self._copy_ms_meas > 1.02 * self._compute_ms)
        if want_zero_copy == self._last_zero_copy:
            self._votes = 0
        else:
            self._votes += 1
            if self._votes >= self.SWITCH_VOTES:
                self._last_zero_copy = want_zero_copy
                self._votes = 0
        return self._last_zero_copy

    def flush(self):
        """Compute the last pending step; returns its results-ready event (or None)."""
        prev, self._pending = self._pending, None
        done = self._compute(prev) if prev is not None else None
        self._burst += 1  # a period across this point would span the caller's idle time
        return done

    def close(self):
        """Restore a passed-in engine's K2 residency cap and release the extra engines."""
        if self._caller_cap is not None:
            self.engines[0].plan.set_k2_ctas_per_sm(self._caller_cap)
        for e_ in self.engines[1:]:
            e_.plan.close()

    def wait_all(self, stream):
        """Make `stream` wait for every result copy issued so far."""
        for ev in self._out_free:
            if ev is not None:
                stream.wait_event(ev)
