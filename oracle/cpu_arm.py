"""CPU arm of bench.py -- TEST / MEASUREMENT INFRASTRUCTURE ONLY (see oracle/__init__.py).

Times the reference algorithm of the hot path on the host cores: the four ★ stages of
compensate_frame (pipeline.py:117-124 rasterize_weights / accumulate_view / solve_view per view,
:79-86 update_all), as restated in oracle/ (C raster + accumulate, numpy/LAPACK solve and fuse,
pinned against the reference's own outputs by tests/test_oracle_*.py).  One process per host
core (fork, BLAS limited to one thread per process): a step is one whole frame, every view's
raster -> accumulate -> solve as one task, then update_all over Gaussian slices -- the
reference's per-frame process pool (pipeline.py:154) applied to views and Gaussian slices.

Inputs come from the oracle tracker (oracle.oracle_track, scene.py:192-240) in the same pool, so
nothing here loads the repo's CUDA library.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

import oracle

_S = {}  # fork-inherited state of the pool workers


def _shared(shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = mp.RawArray("b", max(n, 1))
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def _init_worker():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:  # pragma: no cover
        pass


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    return len(os.sched_getaffinity(0))


# ---------------------------------------------------------------------------------------------
# tracks

def _track_task(v):
    s = _S
    t0 = time.process_time()
    wm = oracle.rasterize(s["g0"], s["cams"][v])
    tgt, val = oracle.oracle_track(s["g0"], s["gt"], s["cams"][v], wm, v, s["frame"],
                                   s["noise"], s["seed"], rel=s["rel"])
    s["tgt"][v] = tgt.astype("<f4")  # TRKF layout (fileio.py:111-136)
    s["val"][v] = val
    return time.process_time() - t0


def oracle_tracks(frame0, frame_t, cams, target_frame, procs=None, noise_sigma_px=0.0, seed=0):
    """Dense tracks of every view (scene.py:192-240 via oracle.oracle_track), TRKF float32.
    Returns (target (V,H,W,2) float32, valid (V,H,W) uint8)."""
    cams = np.asarray(cams, np.float64)
    nv = len(cams)
    w, h = int(cams[0, 16]), int(cams[0, 17])
    _S.clear()
    _S.update(g0=np.ascontiguousarray(frame0), gt=np.ascontiguousarray(frame_t), cams=cams,
              frame=target_frame, noise=noise_sigma_px, seed=seed,
              rel=oracle.relative_rotations(frame0, frame_t),
              tgt=_shared((nv, h, w, 2), np.float32), val=_shared((nv, h, w), np.uint8))
    with mp.get_context("fork").Pool(min(procs or host_cores(), nv), _init_worker) as pool:
        list(pool.imap_unordered(_track_task, range(nv)))
    return np.array(_S["tgt"]), np.array(_S["val"])


# ---------------------------------------------------------------------------------------------
# the timed frame

def _view_task(v):
    s = _S
    t0 = time.process_time()
    wm = oracle.rasterize(s["g"], s["cams"][v], s["cfg"]["alpha_cutoff"])
    acc = oracle.accumulate(wm, s["tgt"][v], s["val"][v], s["n"], s["cfg"]["static_threshold_px"])
    sv = oracle.solve_view(acc, s["cfg"]["det_floor"], s["cfg"]["min_pixels"],
                           s["cfg"]["min_weight"])
    for k in ("status", "a", "b", "weight_sum", "pixel_count"):
        s["mot"][k][v] = sv[k]
    return time.process_time() - t0


def _fuse_task(sl):
    s = _S
    lo, hi = sl
    t0 = time.process_time()
    sub = {k: s["mot"][k][:, lo:hi] for k in s["mot"]}
    c = s["cfg"]
    u = oracle.update_all(s["g"][lo:hi], sub, s["cams"], c["min_views"], c["min_total_weight"],
                          c["min_total_pixels"], c["eig_floor"])
    for k in ("delta_mean", "rotation", "scale", "status"):
        s["upd"][k][lo:hi] = u[k]
    return time.process_time() - t0


class CpuFrame:
    """A process pool holding one frame's inputs; `step()` runs the whole ★ path once."""

    CFG = dict(alpha_cutoff=1.0 / 255.0, det_floor=1e-12, min_pixels=3, min_weight=1e-3,
               min_views=2, min_total_weight=1e-3, min_total_pixels=3, static_threshold_px=1.0,
               eig_floor=1e-12)

    def __init__(self, gaussians, cams, targets, valids, procs=None):
        g = np.ascontiguousarray(gaussians, np.float64)
        cams = np.asarray(cams, np.float64)
        n, nv = len(g), len(cams)
        self.n, self.nv = n, nv
        self.procs = procs or host_cores()
        mot = dict(status=_shared((nv, n), np.int8), a=_shared((nv, n, 2, 2), np.float64),
                   b=_shared((nv, n, 2), np.float64), weight_sum=_shared((nv, n), np.float64),
                   pixel_count=_shared((nv, n), np.int64))
        upd = dict(delta_mean=_shared((n, 3), np.float64), rotation=_shared((n, 4), np.float64),
                   scale=_shared((n, 3), np.float64), status=_shared((n,), np.int8))
        _S.clear()
        _S.update(g=g, cams=cams, n=n, cfg=self.CFG, mot=mot, upd=upd,
                  tgt=[np.asarray(t, np.float64) for t in targets],
                  val=[np.asarray(v, bool) for v in valids])
        self.mot, self.upd = mot, upd
        nsl = 4 * self.procs
        edges = np.linspace(0, n, nsl + 1).astype(int)
        self.slices = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]
        self.pool = mp.get_context("fork").Pool(self.procs, _init_worker)

    def step(self):
        """One frame: returns (wall seconds, summed single-process CPU seconds)."""
        t0 = time.perf_counter()
        cpu = sum(self.pool.imap_unordered(_view_task, range(self.nv)))
        cpu += sum(self.pool.imap_unordered(_fuse_task, self.slices))
        return time.perf_counter() - t0, cpu

    def tallies(self):
        st = np.asarray(self.upd["status"])
        return {"solved": int((st == 1).sum()), "unsolvable": int((st != 1).sum())}

    def close(self):
        self.pool.close()
        self.pool.join()
        _S.clear()
