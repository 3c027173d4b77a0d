"""Frame sharding across GPUs (one process per GPU, torch.distributed over NCCL).

The hot path shards by independent units: in short-clip mode every target frame depends only on
the clip's first-frame Gaussians and its own tracks (pipeline.py:64-65, :177-222; the paper runs
"subsequent frames in parallel using 1, 2, 4, or 8 GPUs").  So:

  * target frame f of a clip goes to rank (f - first - 1) mod world (round robin);
  * the frame-1 Gaussians are broadcast from rank 0 once per clip (NCCL broadcast);
  * every rank bins the first frame itself (cheaper than shipping sorted lists, and it mirrors the
    weight-map reuse of pipeline.py:191-196), builds the clip's kNN, and runs K2-K4 plus the
    regularisation kernels for its frames;
  * updated Gaussian rows are gathered to rank 0 (NCCL gather).

There is no other data-path collective.  The per-frame arithmetic does not depend on the world
size, so results are bit-identical across GPU counts (the analogue of acceptance criterion C8,
tests/test_acceptance.py:349-363); tests/test_distributed.py checks this with gloo on CPU.
"""

from __future__ import annotations

import numpy as np


def frames_for_rank(target_frames, rank, world):
    """Round-robin assignment of a clip's target frames to ranks."""
    return [f for i, f in enumerate(target_frames) if i % world == rank]


def collective_device(group=None):
    """The device collectives of `group` run on: the current CUDA device for NCCL (which cannot
    move host tensors), the CPU otherwise (gloo)."""
    import torch
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_rows(rows, group=None, src=0, device=None):
    """Broadcast the (N, 11) float64 Gaussian rows of the clip's first frame from `src`
    (on `device`, default: the group's collective device)."""
    import torch
    import torch.distributed as dist
    t = rows if isinstance(rows, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(rows))
    if device is None and dist.is_initialized():
        device = collective_device(group)
    if device is not None:
        t = t.to(device)
    t = t.contiguous()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        shape = torch.tensor(list(t.shape), dtype=torch.int64, device=t.device)
        dist.broadcast(shape, src, group=group)
        if tuple(shape.tolist()) != tuple(t.shape):
            t = torch.empty(tuple(shape.tolist()), dtype=torch.float64, device=t.device)
        dist.broadcast(t, src, group=group)
    return t


def gather_frames(local, n_rows, target_frames, group=None, dst=0):
    """Gather {frame: (N, 11) rows} from every rank to `dst`; returns {frame: rows} on dst
    (ordered by frame) and None elsewhere.  Ranks own frames round robin (frames_for_rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return {f: local[f] for f in sorted(local)}
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per_rank = [frames_for_rank(target_frames, r, world) for r in range(world)]
    slots = max(len(p) for p in per_rank)
    # every rank (including one that owns no frame) uses the group's collective device
    device = collective_device(group)
    buf = torch.zeros((slots, n_rows, 11), dtype=torch.float64, device=device)
    for i, f in enumerate(per_rank[rank]):
        buf[i] = torch.as_tensor(local[f]).to(device)
    out = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, out, dst=dst, group=group)
    if rank != dst:
        return None
    result = {}
    for r in range(world):
        for i, f in enumerate(per_rank[r]):
            result[f] = out[r][i]
    return {f: result[f] for f in sorted(result)}


def apply_rows(rows, delta, rotation, scale, status):
    """Updated Gaussian rows (apply_updates semantics, regularize.py:179-188) as tensor ops."""
    import torch
    # torch.where instead of boolean indexing: no device->host sync (a masked index is a nonzero)
    keep = (status != 0)[:, None]
    upd = torch.cat([rows[:, 0:3] + delta, rotation, scale, rows[:, 10:]], 1)
    return torch.where(keep, upd, rows)


def compensate_clip_sharded(first_rows, cameras, tracks_by_frame, target_frames, config=None,
                            group=None, engine=None, compute=None):
    """Compensate every target frame of a short clip across the ranks of `group`.

    tracks_by_frame: {frame: (target, valid)} for (at least) this rank's frames.
    compute(rows, cameras, target, valid) -> updated rows; defaults to the fused GPU engine.
    Returns {frame: updated (N, 11) rows} on rank 0, None on the other ranks.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    rows = broadcast_rows(first_rows, group)
    if compute is None:
        from .config import Config
        from .engine import FrameEngine
        from .regularize import knn_device, regularize_device
        cfg = config or Config()
        eng = engine or FrameEngine()
        eng.bin(rows, cameras, cfg)
        adj = knn_device(eng._gauss, cfg.knn_k)  # once per clip (pipeline.py:197)

        def compute(r, cams, target, valid):
            out = eng.compensate(target, valid)
            return regularize_device(eng._gauss, out.delta_mean, out.rotation, out.scale,
                                     out.status, out.pixel_count, out.static_pixel_count,
                                     eng.n_views, adj, cfg)[5]
    local = {}
    for f in frames_for_rank(target_frames, rank, world):
        target, valid = tracks_by_frame[f]
        local[f] = compute(rows, cameras, target, valid)
    return gather_frames(local, rows.shape[0], target_frames, group)
