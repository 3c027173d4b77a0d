"""On-disk formats of the reference (gausstrack/fileio.py:21-169), array-native.

Formats (byte-compatible with the reference; tests/test_fileio.py reads and writes both ways):
  GAUSS3D  text, header ``GAUSS3D v1 <N>``, one line of 11 ``%.17g`` values per Gaussian
           (mean, quaternion w x y z, scale, opacity)                         fileio.py:24-46
  CAMERA   text, header ``CAMERA v1``, one line of 18 values per camera
           (R row-major, t, fx fy cx cy, width height)                        fileio.py:49-75
  TRACKFIELD text, header ``TRACKFIELD v1 <view> <W> <H>``, one ``x y valid`` row per pixel
                                                                              fileio.py:78-105
  TRKF     binary: ``TRKF`` + little-endian uint32 view, W, H, float32 targets (H, W, 2),
           uint8 validity plane (H, W)                                        fileio.py:108-136

Differences by design: Gaussian sets load into one (N, 11) float64 array wrapped as a lazy
`GaussianList` (no per-Gaussian objects), scenes load as `scene.SceneArrays`, and
`load_trkf_batch` reads V TRKF files straight into one page-locked (V, H, W, 2) float32 +
(V, H, W) uint8 pair -- the layout K2 consumes -- so `upload_tracks` is a single asynchronous
H2D copy per plane.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .core import CameraView, gaussians_array
from .errors import MalformedFile
from .motion2d import TrackField

_FMT = "%.17g"
TRKF_MAGIC = b"TRKF"
_TRKF_HEADER = struct.Struct("<4sIII")


def _rows_text(fh, rows):
    if len(rows):
        np.savetxt(fh, rows, fmt=_FMT, delimiter=" ")


def _parse_rows(lines, width, path, what):
    tokens = []
    for line in lines:
        vals = line.split()
        if len(vals) != width:
            raise MalformedFile(f"{path}: expected {width} values per {what}")
        tokens.extend(vals)
    return np.array(tokens, dtype=np.float64).reshape(-1, width)


# -- GAUSS3D -----------------------------------------------------------------------------------

def save_gaussians(path, gaussians):
    """Write a Gaussian set (list of Gaussian3D, GaussianList or (N, 11) rows)."""
    rows = gaussians_array(gaussians)
    with open(path, "w") as fh:
        fh.write(f"GAUSS3D v1 {len(rows)}\n")
        _rows_text(fh, rows)


def load_gaussian_rows(path):
    """(N, 11) float64 rows of a GAUSS3D file."""
    try:
        with open(path) as fh:
            head = fh.readline().split()
            if len(head) != 3 or head[0] != "GAUSS3D" or head[1] != "v1":
                raise MalformedFile(f"{path}: bad GAUSS3D header")
            count = int(head[2])
            lines = fh.read().splitlines()[:count]
            lines += [""] * (count - len(lines))
            rows = _parse_rows(lines, 11, path, "line")
        # Gaussian3D.__post_init__ (core.py:95-106): validate, renormalise the quaternion
        if not np.all(rows[:, 7:10] > 0):
            raise MalformedFile(f"{path}: scale must be strictly positive")
        if not np.all((rows[:, 10] > 0) & (rows[:, 10] <= 1)):
            raise MalformedFile(f"{path}: opacity must be in (0, 1]")
        from .scene import _normalize_rows
        rows[:, 3:7] = _normalize_rows(rows[:, 3:7])
        return rows
    except (ValueError, OSError) as exc:
        raise MalformedFile(f"{path}: {exc}") from exc


def load_gaussians(path):
    from .pipeline import GaussianList
    return GaussianList(load_gaussian_rows(path))


# -- CAMERA ------------------------------------------------------------------------------------

def save_cameras(path, cameras):
    with open(path, "w") as fh:
        fh.write("CAMERA v1\n")
        for c in cameras:
            vals = list(c.rotation.ravel()) + list(c.translation) + [c.fx, c.fy, c.cx, c.cy,
                                                                     c.width, c.height]
            fh.write(" ".join(_FMT % x for x in vals) + "\n")


def load_cameras(path):
    try:
        with open(path) as fh:
            if fh.readline().split() != ["CAMERA", "v1"]:
                raise MalformedFile(f"{path}: bad CAMERA header")
            rows = _parse_rows([ln for ln in fh if ln.strip()], 18, path, "camera")
        return [CameraView(r[:9].reshape(3, 3), r[9:12], r[12], r[13], r[14], r[15],
                           int(r[16]), int(r[17])) for r in rows]
    except (ValueError, OSError) as exc:
        raise MalformedFile(f"{path}: {exc}") from exc


# -- TRACKFIELD (text) -------------------------------------------------------------------------

def save_trackfield_text(path, tf: TrackField):
    with open(path, "w") as fh:
        fh.write(f"TRACKFIELD v1 {tf.view_id} {tf.width} {tf.height}\n")
        flat = tf.target.reshape(-1, 2)
        valid = tf.valid.reshape(-1)
        for (x, y), ok in zip(flat, valid):
            fh.write(f"{_FMT % x} {_FMT % y} {1 if ok else 0}\n")


def load_trackfield_text(path) -> TrackField:
    try:
        with open(path) as fh:
            head = fh.readline().split()
            if len(head) != 5 or head[0] != "TRACKFIELD" or head[1] != "v1":
                raise MalformedFile(f"{path}: bad TRACKFIELD header")
            view_id, w, h = (int(x) for x in head[2:])
            data = np.loadtxt(fh, ndmin=2)
        if data.shape != (w * h, 3):
            raise MalformedFile(f"{path}: expected {w * h} rows")
        return TrackField(view_id, w, h, data[:, :2].reshape(h, w, 2),
                          data[:, 2].reshape(h, w) != 0)
    except (ValueError, OSError) as exc:
        raise MalformedFile(f"{path}: {exc}") from exc


# -- TRKF (binary) -----------------------------------------------------------------------------

def save_trackfield_binary(path, tf: TrackField):
    with open(path, "wb") as fh:
        fh.write(_TRKF_HEADER.pack(TRKF_MAGIC, tf.view_id, tf.width, tf.height))
        fh.write(np.ascontiguousarray(tf.target, dtype="<f4").tobytes())
        fh.write(np.ascontiguousarray(tf.valid, dtype=np.uint8).tobytes())


def save_trkf_arrays(path, view_id, target, valid):
    """Write one view of the (H, W, 2) float32 / (H, W) uint8 device-layout planes as TRKF."""
    target = np.ascontiguousarray(target, dtype="<f4")
    h, w = target.shape[:2]
    with open(path, "wb") as fh:
        fh.write(_TRKF_HEADER.pack(TRKF_MAGIC, view_id, w, h))
        fh.write(target.tobytes())
        fh.write(np.ascontiguousarray(valid, dtype=np.uint8).tobytes())


def _trkf_header(fh, path):
    if fh.read(4) != TRKF_MAGIC:
        raise MalformedFile(f"{path}: bad TRKF magic")
    raw = fh.read(12)
    if len(raw) != 12:
        raise MalformedFile(f"{path}: truncated TRKF header")
    return struct.unpack("<III", raw)


def _read_exact(fh, buf, what, path):
    if fh.readinto(buf) != buf.nbytes:
        raise MalformedFile(f"{path}: truncated {what}")


def load_trackfield_binary(path) -> TrackField:
    try:
        with open(path, "rb") as fh:
            view_id, w, h = _trkf_header(fh, path)
            tgt = np.empty((h, w, 2), dtype="<f4")
            val = np.empty((h, w), dtype=np.uint8)
            _read_exact(fh, tgt.reshape(-1).view(np.uint8), "target block", path)
            _read_exact(fh, val.reshape(-1), "validity plane", path)
        return TrackField(view_id, w, h, tgt.astype(np.float64), val != 0)
    except (ValueError, OSError, struct.error) as exc:
        raise MalformedFile(f"{path}: {exc}") from exc


def load_trkf_batch(paths, pinned=True):
    """Read V TRKF files into one (V, H, W, 2) float32 + (V, H, W) uint8 host tensor pair,
    page-locked when `pinned` and CUDA is available.  Returns (target, valid, view_ids).

    Targets stay float32 as stored (K2 reads TS_TRACK_F32 tracks directly); the reference widens
    them to float64 on load, which is exact, so the results are the same.
    """
    import torch
    if not paths:
        raise MalformedFile("load_trkf_batch: no files")
    target = valid = None
    ids = []
    for v, path in enumerate(paths):
        try:
            with open(path, "rb") as fh:
                view_id, w, h = _trkf_header(fh, path)
                if target is None:
                    pin = pinned and torch.cuda.is_available()
                    target = torch.empty((len(paths), h, w, 2), dtype=torch.float32,
                                         pin_memory=pin)
                    valid = torch.empty((len(paths), h, w), dtype=torch.uint8, pin_memory=pin)
                elif tuple(target.shape[1:3]) != (h, w):
                    raise MalformedFile(f"{path}: views disagree on image size")
                _read_exact(fh, target[v].numpy().reshape(-1).view(np.uint8), "target block",
                            path)
                _read_exact(fh, valid[v].numpy().reshape(-1), "validity plane", path)
                ids.append(view_id)
        except (ValueError, OSError, struct.error) as exc:
            raise MalformedFile(f"{path}: {exc}") from exc
    return target, valid, ids


def upload_tracks(target, valid, stream=None):
    """Asynchronous H2D copy of a (pinned) track batch; returns the device tensors.  Ordered on
    `stream` (default: the current stream)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        t_d = torch.empty(target.shape, dtype=target.dtype, device="cuda")
        v_d = torch.empty(valid.shape, dtype=torch.uint8, device="cuda")
        t_d.copy_(target, non_blocking=True)
        v_d.copy_(valid, non_blocking=True)
    return t_d, v_d


# -- scene directories (fileio.py:142-169) -----------------------------------------------------

def frame_filename(frame):
    return f"frame_{frame:04d}.txt"


def track_filename(view, frame):
    return f"track_view{view:03d}_frame{frame:04d}.trk"


def save_scene(dirpath, scene):
    """cameras.txt + one GAUSS3D file per frame (scene: SceneArrays or the reference's
    SceneSequence -- anything with .cameras and .frames)."""
    os.makedirs(dirpath, exist_ok=True)
    save_cameras(os.path.join(dirpath, "cameras.txt"), scene.cameras)
    for t, frame in enumerate(scene.frames):
        save_gaussians(os.path.join(dirpath, frame_filename(t)), frame)


def load_scene(dirpath):
    """SceneArrays of a scene directory (no per-frame ground-truth motion, like the reference)."""
    from .scene import SceneArrays
    cameras = load_cameras(os.path.join(dirpath, "cameras.txt"))
    frames = []
    while os.path.exists(os.path.join(dirpath, frame_filename(len(frames)))):
        frames.append(load_gaussian_rows(os.path.join(dirpath, frame_filename(len(frames)))))
    if not frames:
        raise MalformedFile(f"{dirpath}: no frame files found")
    if len({len(f) for f in frames}) != 1:
        raise MalformedFile(f"{dirpath}: frames disagree on Gaussian count")
    return SceneArrays(cameras, frames, None, None)
