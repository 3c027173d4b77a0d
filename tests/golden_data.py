"""Loaders for the reference-generated fixtures in tests/golden/ (see make_golden.py)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def tracks(d):
    """Rebuild dense (V,H,W,2) float64 targets and (V,H,W) bool valid masks; invalid pixels
    carry identity targets as oracle_track leaves them (scene.py:213-214)."""
    shape = tuple(int(s) for s in d["track_shape"])
    valid = np.unpackbits(d["track_valid_bits"])[: int(np.prod(shape))].reshape(shape).astype(bool)
    v, h, w = shape
    ys, xs = np.mgrid[0:h, 0:w]
    target = np.broadcast_to(np.stack([xs, ys], -1).astype(np.float64), (v, h, w, 2)).copy()
    target[valid] = d["track_target_valid"].astype(np.float64)
    return target, valid


def weightmap(d, prefix):
    return dict(pixel_x=d[prefix + "px"].astype(np.int32), pixel_y=d[prefix + "py"].astype(np.int32),
                gaussian_id=d[prefix + "gid"].astype(np.int64), alpha=d[prefix + "alpha"],
                transmittance=d[prefix + "trans"], degenerate_ids=d[prefix + "deg"])


def motions(d):
    return dict(status=d["m_status"], a=d["m_a"], b=d["m_b"], weight_sum=d["m_w"],
                pixel_count=d["m_cnt"])


def tile_order_index(ranges):
    """Instance indices of one view's tiles in tile order, from its (tiles, 2) [start, end)
    ranges (empty tiles contribute nothing)."""
    ranges = np.asarray(ranges, np.int64)
    cnt = ranges[:, 1] - ranges[:, 0]
    if not cnt.any():
        return np.zeros(0, np.int64)
    starts = np.repeat(ranges[:, 0], cnt)
    within = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    return starts + within
