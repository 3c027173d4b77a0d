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


TRACKER_SCENES = {  # tracker_kats.npz cases: generate_scene args / kwargs (make_golden.py)
    "dom": ((2, 20, 4, 2), {}),
    "static": ((4, 30, 4, 3), dict(mover_fraction=0.0)),
    "cover": ((4, 30, 4, 3), {}),
    "noisy": ((4, 30, 4, 3), {}),
    "transl": ((6, 40, 4, 2), dict(mover_fraction=1.0, translate_mag=0.03, rotate_deg=0.0)),
}

# the scene fixtures with reference tracks: generate_scene args / kwargs, noise sigma
SCENE_TRACKS = {
    "scene21": ((21, 120, 4, 2), dict(mover_fraction=0.25, translate_mag=0.02), 0.0),
    "scene7": ((7, 2000, 8, 2), dict(mover_fraction=0.3, translate_mag=0.02, rotate_deg=2.0), 0.5),
    "cfg1": ((1, 10_000, 4, 2), dict(focal=180, width=128, height=128, scale_range=(0.01, 0.02)),
             0.0),
}


def tracker_case(d, tag):
    """(meta dict, per-view dict of reference dominant gid / depth images and tracks)."""
    view, frame, noise, seed = d[f"{tag}_meta"]
    cams = d[f"{tag}_cameras"]
    w, h = int(cams[0, 16]), int(cams[0, 17])
    views = range(len(cams)) if view < 0 else [int(view)]
    out = {}
    for v in views:
        valid = np.unpackbits(d[f"{tag}_v{v}_valid_bits"])[: w * h].reshape(h, w).astype(bool)
        ys, xs = np.mgrid[0:h, 0:w]
        target = np.stack([xs, ys], -1).astype(np.float64)
        target[valid] = d[f"{tag}_v{v}_target_valid"]
        out[v] = dict(gid=d[f"{tag}_v{v}_dom_gid"].astype(np.int64),
                      depth=d[f"{tag}_v{v}_dom_depth"], target=target, valid=valid)
    meta = dict(frame=int(frame), noise=float(noise), seed=int(seed), cameras=cams,
                g0=d[f"{tag}_gaussians0"], g1=d[f"{tag}_gaussians1"])
    return meta, out
