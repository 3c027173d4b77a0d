"""Motion-compensation entry point (gausstrack/pipeline.py:32-129) on the fused GPU path.

`compensate_frame` keeps the reference signature.  Its four hot-path stages (rasterize,
accumulate, per-view solve, multi-view fuse: pipeline.py:117-124 and :79-86) run as
K1 -> K2 -> K3 -> K4 on the device without materialising weight maps or per-view objects, and
the regularisation tail (static flags, kNN median filter, propagation, apply_updates:
pipeline.py:88-98, regularize.py:37-188) runs as two more kernels on the K4 outputs
(regularize.regularize_device), with the exact kNN built on the device when `knn` is None.
`regularize=False` returns the K4 updates unregularised; a callable
`regularize(frame1, updates, accs, config, knn) -> updates` replaces the stage (e.g.
tools/reference_regularizer.py, which wraps the reference's CPU implementation for
cross-checks; the product package never runs reference code).
"""

from __future__ import annotations

import csv
import io
import time
from dataclasses import dataclass, field

import numpy as np

from .config import Config
from .core import Gaussian3D, cameras_array, gaussians_array
from .errors import DimensionMismatch, InvalidConfig
from .motion2d import ViewAccumulators
from .multiview import MotionUpdateList


@dataclass(frozen=True)
class Clip:
    first_frame: int
    target_frames: tuple
    views: tuple


@dataclass
class FrameResult:
    frame: int
    gaussians: list
    tallies: dict
    wall_time: dict
    compensated_from: int | None = None


class GaussianList:
    """Array-backed, lazily materialised list[Gaussian3D] (rows: (N, 11) float64)."""

    def __init__(self, rows):
        self.rows = np.ascontiguousarray(rows, np.float64).reshape(-1, 11)

    def __len__(self):
        return len(self.rows)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        r = self.rows[i]
        return Gaussian3D(r[0:3], r[3:7], r[7:10], r[10])

    def __iter__(self):
        return (self[i] for i in range(len(self)))


def segment_clips(n_frames, clip_len, n_views, mode="short"):
    """Short mode: disjoint blocks re-seeded from ground truth; long mode: chained blocks
    sharing boundary frames (pipeline.py:48-72)."""
    if clip_len < 2:
        raise InvalidConfig(f"clip_len must be >= 2, got {clip_len}")
    if mode not in ("short", "long"):
        raise InvalidConfig(f"mode must be short|long, got {mode!r}")
    views = tuple(range(n_views))
    clips = []
    if mode == "short":
        for first in range(0, n_frames, clip_len):
            last = min(first + clip_len, n_frames)
            clips.append(Clip(first, tuple(range(first + 1, last)), views))
        return clips
    first = 0
    while first < n_frames - 1:
        last = min(first + clip_len - 1, n_frames - 1)
        clips.append(Clip(first, tuple(range(first + 1, last + 1)), views))
        first = last
    return clips


def apply_update_rows(rows, delta, rotation, scale, status):
    """apply_updates (regularize.py:179-188) on arrays: unsolvable rows keep frame-1 values."""
    out = np.array(rows, np.float64, copy=True).reshape(-1, 11)
    keep = np.asarray(status) != 0
    out[keep, 0:3] += delta[keep]
    out[keep, 3:7] = rotation[keep]
    out[keep, 7:10] = scale[keep]
    return out


def _tracks_arrays(tracks, n_views):
    """Stack TrackField objects (or pass (V,H,W,2)/(V,H,W) arrays through)."""
    if isinstance(tracks, tuple) and len(tracks) == 2:
        return tracks
    if len(tracks) != n_views:
        raise DimensionMismatch("track fields and cameras count differ")
    if len({(t.width, t.height) for t in tracks}) > 1:
        # per-view image sizes (pipeline.py:117-120): per-view lists, FrameEngine bins size groups
        tgts, vals = [], []
        for t in tracks:
            tg = np.asarray(t.target)
            va = np.asarray(t.valid, bool)
            if np.all(tg[va] == tg[va].astype(np.float32)):
                tg = tg.astype(np.float32)
            tgts.append(tg)
            vals.append(va.astype(np.uint8))
        return tgts, vals
    target = np.stack([np.asarray(t.target) for t in tracks])
    valid = np.stack([np.asarray(t.valid, bool) for t in tracks]).astype(np.uint8)
    if np.all(target[valid.astype(bool)] == target[valid.astype(bool)].astype(np.float32)):
        target = target.astype(np.float32)  # TRKF-exact values: ship 4-byte targets
    return target, valid


_ENGINES = {}


def _engine():
    import torch

    from .engine import FrameEngine
    dev = torch.cuda.current_device()
    if dev not in _ENGINES:
        _ENGINES[dev] = FrameEngine()
    return _ENGINES[dev]


def _knn_adjacency(knn, rows_dev, config):
    import torch

    from .regularize import knn_device
    if knn is None:
        return knn_device(rows_dev, config.knn_k)
    adj = np.asarray(knn.adjacency if hasattr(knn, "adjacency") else knn, np.int64)
    return torch.from_numpy(adj.reshape(len(adj), -1)).to(rows_dev.device)


def _result(frame_index, first_frame_index, new_rows, status, t0):
    st = np.asarray(status)
    tallies = {"solved": int((st == 1).sum()), "static": int((st == 2).sum()),
               "unsolvable": int((st == 0).sum())}
    return FrameResult(frame_index, GaussianList(new_rows), tallies,
                       {"tracking": 0.0, "compensation": time.perf_counter() - t0,
                        "refinement": 0.0}, compensated_from=first_frame_index)


def compensate_frame(frame1, cameras, tracks, config: Config = None, weightmaps=None, knn=None,
                     frame_index=0, first_frame_index=0, regularize=True) -> FrameResult:
    """Full single-frame motion compensation from first-frame Gaussians and per-view tracks.

    Without `weightmaps` this is the fused GPU path (K1-K4 + regularisation); with them it runs
    the GPU stage kernels on the given weight maps (as the reference skips its rasterizer).
    """
    import torch

    from .regularize import regularize_device
    config = config or Config()
    t0 = time.perf_counter()
    rows = gaussians_array(frame1)
    cams = cameras_array(cameras)
    n, nv = len(rows), len(cams)
    if weightmaps is None:
        eng = _engine()
        eng.bin(rows, cams, config)
        target, valid = _tracks_arrays(tracks, nv)
        out = eng.compensate(target, valid)
        g_dev = eng._gauss
        k4 = (out.delta_mean, out.rotation, out.scale, out.status)
        pc_dev, sc_dev = out.pixel_count, out.static_pixel_count
        accs = None
        if callable(regularize):
            torch.cuda.synchronize()
            mc = out.pixel_count.cpu().numpy().reshape(nv, n).astype(np.int64)
            msc = out.static_pixel_count.cpu().numpy().reshape(nv, n).astype(np.int64)
            msw = out.static_weight_sum.cpu().numpy().reshape(nv, n)
            mw = out.weight_sum.cpu().numpy().reshape(nv, n)
            accs = [ViewAccumulators(v, None, None, mw[v], mc[v], msc[v], msw[v])
                    for v in range(nv)]
    else:
        from .engine import as_device
        from .motion2d import accumulate_view, solve_view
        from .multiview import update_all
        accs = [accumulate_view(wm, tf, n, config.static_threshold_px)
                for wm, tf in zip(weightmaps, tracks)]
        motions = [solve_view(a, config.det_floor, config.min_pixels, config.min_weight)
                   for a in accs]
        upd = update_all(rows, motions, cams, config.min_views, config.min_total_weight,
                         config.min_total_pixels, config.eig_floor)
        g_dev = as_device(rows, torch.float64)
        k4 = (as_device(upd.delta_mean, torch.float64), as_device(upd.rotation, torch.float64),
              as_device(upd.scale, torch.float64), as_device(upd.status, torch.int8))
        pc_dev = as_device(np.stack([a.pixel_count for a in accs]).astype(np.int32), torch.int32)
        sc_dev = as_device(np.stack([a.static_pixel_count for a in accs]).astype(np.int32),
                           torch.int32)
    if callable(regularize):
        updates = MotionUpdateList(*(t.cpu().numpy() for t in k4))
        updates = regularize(frame1, updates, accs, config, knn)
        k4 = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(g_dev.device)
                   for a in (updates.delta_mean, updates.rotation, updates.scale,
                             np.asarray(updates.status, np.int8)))
        regularize = False
    if regularize:
        adj = _knn_adjacency(knn, g_dev, config)
        *_, status, _flags, new_rows = regularize_device(g_dev, *k4, pc_dev, sc_dev, nv, adj,
                                                         config)
    else:
        from .regularize import apply_rows_device
        status = k4[3]
        new_rows = apply_rows_device(g_dev, *k4)
    return _result(frame_index, first_frame_index, new_rows.cpu().numpy(), status.cpu().numpy(),
                   t0)


# -- clip driver (pipeline.py:132-237) -----------------------------------------------------------

def _scene_arrays(scene):
    """SceneArrays view of our SceneArrays or the reference's SceneSequence (object frames)."""
    from .scene import SceneArrays
    if isinstance(scene, SceneArrays):
        return scene
    frames = [gaussians_array(f) for f in scene.frames]
    return SceneArrays(list(scene.cameras), frames, None, None)


def _zero_result(frame, rows):
    return FrameResult(frame, GaussianList(rows), {"solved": 0, "static": 0, "unsolvable": 0},
                       {"tracking": 0.0, "compensation": 0.0, "refinement": 0.0})


def _share_clip_results(results, clip, n, group):
    """All-gather the FrameResults of a clip's target frames (rows over NCCL, metadata as
    objects); each frame is owned by one rank (distributed.frames_for_rank)."""
    import torch
    import torch.distributed as dist

    from .distributed import frames_for_rank
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per_rank = [frames_for_rank(clip.target_frames, r, world) for r in range(world)]
    slots = max(len(p) for p in per_rank)
    if slots == 0:
        return
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf = torch.zeros((slots, n, 11), dtype=torch.float64, device=dev)
    meta = []
    for i, f in enumerate(per_rank[rank]):
        r = results[f]
        buf[i] = torch.from_numpy(np.ascontiguousarray(r.gaussians.rows)).to(dev)
        meta.append((f, r.tallies, r.wall_time, r.compensated_from))
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    metas = [None] * world
    dist.all_gather_object(metas, meta, group=group)
    for r in range(world):
        for i, (f, tallies, wall, src) in enumerate(metas[r]):
            results[f] = FrameResult(f, GaussianList(bufs[r][i].cpu().numpy()), tallies, wall,
                                     compensated_from=src)


def run_pipeline(scene, clip_len, workers=1, config: Config = None, mode="short",
                 noise_sigma_px=0.0, seed=0, refine_hook=None, stage_totals=None, group=None):
    """Tracking + compensation over every clip of a scene (pipeline.py:132-237) on the GPU.

    Per clip: the tracker's binning of the ground-truth first frame (K1) is reused for the
    compensation when the clip starts from ground truth (short mode, or the first clip of a
    chain) -- the reference's weight-map reuse (:191-196), which also covers the rasterization:
    with several target frames the contributions are cached once per clip (ts_frame_cache); the
    exact kNN is built once per clip on the device; every target frame then runs the GPU oracle
    tracker, K2+K3 from the cache (or K2-K3), K4 and the regularisation kernels.  Long mode chains clips through the previous clip's estimate of its last frame.

    `workers` is accepted for signature parity (>= 1); parallelism comes from the GPU and, when
    torch.distributed is initialised with more than one rank (`group`), from frame sharding:
    target frames are dealt round robin to ranks and every rank ends with the full result list
    (all-gather per clip, so long-mode chains see the previous clip's last frame).  Results do
    not depend on the world size.  stage_totals accumulates setup / tracking / fuse seconds.
    """
    import torch
    import torch.distributed as dist

    from .distributed import frames_for_rank
    from .engine import FrameEngine
    from .regularize import knn_device, regularize_device
    from .scene import oracle_tracks
    if workers < 1:
        raise InvalidConfig(f"workers must be >= 1, got {workers}")
    config = config or Config()
    if stage_totals is None:
        stage_totals = {}
    stage_totals.update({"setup": 0.0, "tracking": 0.0, "fuse": 0.0})
    scene = _scene_arrays(scene)
    cams = cameras_array(scene.cameras)
    nv = len(cams)
    clips = segment_clips(scene.n_frames, clip_len, nv, mode)
    sharded = dist.is_initialized() and dist.get_world_size(group) > 1
    world = dist.get_world_size(group) if sharded else 1
    rank = dist.get_rank(group) if sharded else 0

    results = {0: _zero_result(0, scene.frames[0])}
    eng_track, eng_comp = FrameEngine(), None
    for clip in clips:
        gt_first = scene.frames[clip.first_frame]
        if mode == "short":
            first_rows = gt_first
            results.setdefault(clip.first_frame, _zero_result(clip.first_frame, gt_first))
        else:
            first_rows = results[clip.first_frame].gaussians.rows
        if not clip.target_frames:
            continue
        t0 = time.perf_counter()
        eng_track.bin(gt_first, cams, config)
        if first_rows is gt_first or np.array_equal(first_rows, gt_first):
            eng = eng_track
        else:
            eng_comp = eng_comp or FrameEngine()
            eng = eng_comp.bin(first_rows, cams, config)
        g_dev = eng._gauss
        adj = knn_device(g_dev, config.knn_k)
        mine = frames_for_rank(clip.target_frames, rank, world)
        if len(mine) > 1:
            # the clip's target frames share frame 0's contributions: rasterize once
            # (the reference's weight-map reuse, :191-196) and apply each frame's tracks
            eng.build_cache()
        torch.cuda.synchronize()
        stage_totals["setup"] += time.perf_counter() - t0
        for f in mine:
            t0 = time.perf_counter()
            tgt, val = oracle_tracks(scene, f, noise_sigma_px, seed, first_frame=clip.first_frame,
                                     engine=eng_track)
            torch.cuda.synchronize()
            t_track = time.perf_counter() - t0
            t0 = time.perf_counter()
            out = eng.compensate(tgt, val)
            *_, status, _flags, rows = regularize_device(
                g_dev, out.delta_mean, out.rotation, out.scale, out.status, out.pixel_count,
                out.static_pixel_count, nv, adj, config)
            rows_h, st = rows.cpu().numpy(), status.cpu().numpy()
            t_comp = time.perf_counter() - t0
            res = _result(f, clip.first_frame, rows_h, st, t0)
            res.wall_time.update(tracking=t_track, compensation=t_comp)
            if refine_hook is not None:
                t0 = time.perf_counter()
                res.gaussians = refine_hook(res.frame, res.gaussians)
                res.wall_time["refinement"] = time.perf_counter() - t0
            stage_totals["tracking"] += t_track
            stage_totals["fuse"] += t_comp
            results[f] = res
        if sharded:
            _share_clip_results(results, clip, len(first_rows), group)
    return [results[f] for f in sorted(results)]


# -- evaluation (pipeline.py:243-298) ------------------------------------------------------------

CSV_COLUMNS = ["frame", "mean_pos_err", "p95_pos_err", "mean_rot_err_deg", "mean_rel_scale_err",
               "n_solved", "n_static", "n_unsolvable", "t_track", "t_comp", "t_refine"]


@dataclass
class EvaluationReport:
    rows: list = field(default_factory=list)

    def write_csv(self, path):
        with open(path, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=CSV_COLUMNS)
            w.writeheader()
            w.writerows(self.rows)

    def summary(self):
        out = io.StringIO()
        out.write(f"{'frame':>6} {'pos_err':>12} {'p95_pos':>12} {'rot_deg':>10} "
                  f"{'scale_rel':>10} {'solved':>7} {'static':>7} {'unsolv':>7}\n")
        for r in self.rows:
            out.write(f"{r['frame']:>6} {r['mean_pos_err']:>12.6g} {r['p95_pos_err']:>12.6g} "
                      f"{r['mean_rot_err_deg']:>10.4g} {r['mean_rel_scale_err']:>10.4g} "
                      f"{r['n_solved']:>7} {r['n_static']:>7} {r['n_unsolvable']:>7}\n")
        return out.getvalue()


def _unit_rows(q):
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def evaluate(results, scene) -> EvaluationReport:
    """Ground-truth error per frame: position, rotation (geodesic, degrees), relative scale
    (pipeline.py:273-298), vectorised over the Gaussians."""
    scene = _scene_arrays(scene)
    report = EvaluationReport()
    for res in results:
        est = gaussians_array(res.gaussians)
        truth = scene.frames[res.frame]
        pos_err = np.linalg.norm(est[:, 0:3] - truth[:, 0:3], axis=1)
        d = np.abs(np.sum(_unit_rows(est[:, 3:7]) * _unit_rows(truth[:, 3:7]), axis=1))
        rot_err = 2.0 * np.arccos(np.minimum(d, 1.0))
        scale_err = np.mean(np.abs(est[:, 7:10] - truth[:, 7:10]) / truth[:, 7:10], axis=1)
        report.rows.append({
            "frame": res.frame,
            "mean_pos_err": float(np.mean(pos_err)),
            "p95_pos_err": float(np.percentile(pos_err, 95)),
            "mean_rot_err_deg": float(np.degrees(np.mean(rot_err))),
            "mean_rel_scale_err": float(np.mean(scale_err)),
            "n_solved": res.tallies["solved"],
            "n_static": res.tallies["static"],
            "n_unsolvable": res.tallies["unsolvable"],
            "t_track": res.wall_time["tracking"],
            "t_comp": res.wall_time["compensation"],
            "t_refine": res.wall_time["refinement"],
        })
    return report
