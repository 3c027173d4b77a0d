"""Frame sharding over torch.distributed (gloo, world size 2, CPU).

The per-frame compute is the CPU oracle here (tests only); the sharding, broadcast and gather are
the product code of paper_2604_02586_b200.distributed, which bench.py drives over NCCL on GPUs.
Results must be bit-identical to the single-process run (acceptance criterion C8 analogue,
reference tests/test_acceptance.py:349-363).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2604_02586_b200.distributed import (apply_rows, compensate_clip_sharded,
                                               frames_for_rank)
from paper_2604_02586_b200.scene import generate_scene

TARGETS = (1, 2, 3)


def _scene():
    sc = generate_scene(13, 80, 4, 4)
    cams = np.array([c.as_row() for c in sc.cameras])
    h, w = sc.cameras[0].height, sc.cameras[0].width
    ys, xs = np.mgrid[0:h, 0:w]
    base = np.stack([xs, ys], -1).astype(np.float64)
    tracks = {f: (np.stack([base + np.array([0.35 * f, -0.2 * f])] * 4),
                  np.ones((4, h, w), np.uint8)) for f in TARGETS}
    return sc.frames[0], cams, tracks


def _cpu_compute(rows, cams, target, valid):
    r = rows.numpy()
    upd, _, _ = oracle.compensate(r, cams, list(target), list(valid.astype(bool)))
    return apply_rows(rows, torch.as_tensor(upd["delta_mean"]), torch.as_tensor(upd["rotation"]),
                      torch.as_tensor(upd["scale"]), torch.as_tensor(upd["status"]))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, cams, tracks = _scene()
    # only rank 0 holds the real first frame: the broadcast must deliver it
    first = torch.as_tensor(rows) if rank == 0 else torch.zeros(rows.shape, dtype=torch.float64)
    mine = {f: tracks[f] for f in frames_for_rank(TARGETS, rank, world)}
    res = compensate_clip_sharded(first, cams, mine, TARGETS, compute=_cpu_compute)
    if rank == 0:
        np.savez(out_path, **{str(f): v.numpy() for f, v in res.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_frames_for_rank_partition():
    for world in (1, 2, 3, 4, 8):
        got = sorted(f for r in range(world) for f in frames_for_rank(range(1, 9), r, world))
        assert got == list(range(1, 9))


@pytest.mark.timeout(600)
def test_sharded_equals_serial(tmp_path):
    rows, cams, tracks = _scene()
    serial = {f: _cpu_compute(torch.as_tensor(rows), cams, *tracks[f]).numpy() for f in TARGETS}
    out = tmp_path / "sharded.npz"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    got = np.load(out)
    assert sorted(int(k) for k in got.files) == list(TARGETS)
    for f in TARGETS:
        np.testing.assert_array_equal(got[str(f)], serial[f])
    # the motion actually moved something
    assert np.abs(serial[1][:, 0:3] - rows[:, 0:3]).max() > 0


def _share_worker(rank, world, port, out_path):
    from paper_2604_02586_b200.pipeline import Clip, FrameResult, GaussianList, _share_clip_results
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    clip = Clip(0, (1, 2, 3, 4, 5), (0, 1))
    results = {}
    for f in frames_for_rank(clip.target_frames, rank, world):
        rows = np.full((6, 11), float(f)) + np.arange(11)
        results[f] = FrameResult(f, GaussianList(rows), {"solved": f, "static": 0,
                                                         "unsolvable": 6 - f},
                                 {"tracking": 0.1 * f, "compensation": 0.0, "refinement": 0.0},
                                 compensated_from=0)
    _share_clip_results(results, clip, 6, None)
    np.savez(f"{out_path}.{rank}.npz",
             **{str(f): results[f].gaussians.rows for f in results},
             tallies=np.array([results[f].tallies["solved"] for f in sorted(results)]),
             src=np.array([results[f].compensated_from for f in sorted(results)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_run_pipeline_result_sharing(tmp_path):
    """run_pipeline's per-clip all-gather: every rank ends with every frame (long-mode chains
    need the previous clip's last frame everywhere)."""
    out = str(tmp_path / "share")
    mp.spawn(_share_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for rank in range(2):
        got = np.load(f"{out}.{rank}.npz")
        assert sorted(int(k) for k in got.files if k.isdigit()) == [1, 2, 3, 4, 5]
        for f in range(1, 6):
            np.testing.assert_array_equal(got[str(f)], np.full((6, 11), float(f)) + np.arange(11))
        np.testing.assert_array_equal(got["tallies"], [1, 2, 3, 4, 5])
        np.testing.assert_array_equal(got["src"], [0] * 5)


def _idle_rank_worker(rank, world, port, out_path):
    """world > number of target frames: rank 2 owns none and still joins the gather."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, cams, tracks = _scene()
    first = torch.as_tensor(rows) if rank == 0 else torch.zeros(rows.shape, dtype=torch.float64)
    targets = (1, 2)
    mine = {f: tracks[f] for f in frames_for_rank(targets, rank, world)}
    res = compensate_clip_sharded(first, cams, mine, targets, compute=_cpu_compute)
    if rank == 0:
        np.savez(out_path, **{str(f): v.numpy() for f, v in res.items()})
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_sharded_with_idle_rank(tmp_path):
    rows, cams, tracks = _scene()
    out = tmp_path / "idle.npz"
    mp.spawn(_idle_rank_worker, args=(3, _free_port(), str(out)), nprocs=3, join=True)
    got = np.load(out)
    assert sorted(int(k) for k in got.files) == [1, 2]
    for f in (1, 2):
        serial = _cpu_compute(torch.as_tensor(rows), cams, *tracks[f]).numpy()
        np.testing.assert_array_equal(got[str(f)], serial)
