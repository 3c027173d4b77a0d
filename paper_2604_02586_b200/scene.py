"""Synthetic inputs: the reference scene generator and a GPU oracle tracker.

`generate_scene` restates gausstrack/scene.py:58-163 with the same random-number call sequence,
so it yields the same cameras and first-frame Gaussians as the reference for the same arguments
(pinned by tests/test_scene_generator.py against tests/golden/scenes.npz), but keeps frames as
(N, 11) arrays instead of millions of Python objects.

`oracle_tracks` is the GPU version of oracle_track (scene.py:166-240): the dominant Gaussian of
each pixel (argmax alpha*T, ties by smaller id) comes from K2 in "dominant" mode over the frame-0
binning, the depth-plane transport runs as tensor ops on the device, and the keyed noise is drawn
from the same numpy generator as the reference (default_rng([seed, view, frame])).  It is input
production for benchmarks and large-config parity runs, not part of the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import CameraView, Gaussian3D, quat_multiply, quat_normalize
from .errors import InvalidConfig


@dataclass
class SceneArrays:
    cameras: list             # CameraView
    frames: list              # frames[t]: (N, 11) float64 rows
    step_translation: np.ndarray  # (N, 3) per-frame translation
    step_rotation: np.ndarray     # (N, 4) per-frame quaternion increment

    @property
    def n_frames(self):
        return len(self.frames)

    @property
    def n_gaussians(self):
        return len(self.frames[0])

    def gaussians(self, t):
        return [Gaussian3D(r[0:3], r[3:7], r[7:10], r[10]) for r in self.frames[t]]


def _ring_camera(angle, radius, height, focal, width, img_height):
    position = np.array([radius * np.cos(angle), radius * np.sin(angle), height])
    forward = -position / np.linalg.norm(position)
    right = np.cross(forward, np.array([0.0, 0.0, 1.0]))
    right /= np.linalg.norm(right)
    down = np.cross(forward, right)
    r = np.stack([right, down, forward])
    return CameraView(r, -r @ position, focal, focal, width / 2.0, img_height / 2.0, width,
                      img_height)


def _normalize_rows(q):
    """Row-wise quat_normalize with the reference's scalar numerics (np.linalg.norm per row)."""
    out = np.empty_like(q)
    for i in range(len(q)):
        out[i] = quat_normalize(q[i])
    return out


def generate_scene(seed, n_gaussians, n_views, n_frames, mover_fraction=0.3, translate_mag=0.02,
                   rotate_deg=2.0, scene_radius=1.0, ring_radius=6.0, focal=800.0, width=960,
                   height=540, scale_range=(0.004, 0.008), opacity_range=(0.95, 0.999),
                   check_frustum=True) -> SceneArrays:
    """Ring cameras around a ball of static Gaussians plus a rigidly moving cluster."""
    if n_views < 3:
        raise InvalidConfig(f"need n_views >= 3, got {n_views}")
    if n_gaussians < 10:
        raise InvalidConfig(f"need n_gaussians >= 10, got {n_gaussians}")
    if n_frames < 1:
        raise InvalidConfig("need n_frames >= 1")
    rng = np.random.default_rng(seed)
    cameras = [_ring_camera(2 * np.pi * v / n_views, ring_radius, 0.3 * ring_radius, focal,
                            width, height) for v in range(n_views)]
    n_movers = int(round(mover_fraction * n_gaussians))
    n_static = n_gaussians - n_movers

    def ball(center, radius, count):
        pts = rng.normal(size=(count, 3))
        pts /= np.linalg.norm(pts, axis=1, keepdims=True)
        pts *= radius * rng.uniform(size=(count, 1)) ** (1.0 / 3.0)
        return pts + center

    means = np.empty((n_gaussians, 3))
    means[:n_static] = ball(np.zeros(3), scene_radius, n_static)
    if n_movers:
        angle = rng.uniform(0, 2 * np.pi)
        center = scene_radius * np.array([1.6 * np.cos(angle), 1.6 * np.sin(angle), 0.85])
        means[n_static:] = ball(center, 0.3 * scene_radius, n_movers)
    quats = rng.normal(size=(n_gaussians, 4))
    scales = rng.uniform(*scale_range, size=(n_gaussians, 3))
    opac = rng.uniform(*opacity_range, size=n_gaussians)
    if np.any(scales <= 0) or np.any(opac <= 0) or np.any(opac > 1):
        raise ValueError("invalid scale/opacity range")
    first = np.empty((n_gaussians, 11))
    first[:, 0:3] = means
    first[:, 3:7] = _normalize_rows(quats)
    first[:, 7:10] = scales
    first[:, 10] = opac

    step_t = np.zeros((n_gaussians, 3))
    step_q = np.tile(np.array([1.0, 0.0, 0.0, 0.0]), (n_gaussians, 1))
    if n_movers:
        direction = rng.normal(size=3)
        direction[2] = np.sign(direction[2]) * max(abs(direction[2]), 1.0)
        direction /= np.linalg.norm(direction)
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        half = np.deg2rad(rotate_deg) / 2.0
        q = quat_normalize(np.concatenate([[np.cos(half)], np.sin(half) * axis]))
        step_t[n_static:] = translate_mag * direction
        step_q[n_static:] = q

    frames = [first]
    for _ in range(1, n_frames):
        prev = frames[-1]
        cur = prev.copy()
        cur[:, 0:3] = prev[:, 0:3] + step_t
        # static rows multiply by the identity quaternion; renormalise like Gaussian3D does
        for i in range(n_gaussians):
            cur[i, 3:7] = quat_normalize(quat_multiply(step_q[i], prev[i, 3:7]))
        frames.append(cur)

    if check_frustum:
        for t, frame in enumerate(frames):
            pts = frame[:, 0:3]
            for cam in cameras:
                pc = pts @ cam.rotation.T + cam.translation
                z = pc[:, 2]
                if np.any(z < 0.1 * ring_radius):
                    raise InvalidConfig(f"frame {t}: Gaussians too close to a camera")
                u = cam.fx * pc[:, 0] / z + cam.cx
                v = cam.fy * pc[:, 1] / z + cam.cy
                if (np.any(u < 1) or np.any(u > cam.width - 2) or np.any(v < 1)
                        or np.any(v > cam.height - 2)):
                    raise InvalidConfig(f"frame {t}: Gaussians project outside the image")
    return SceneArrays(cameras, frames, step_t, step_q)


def _quat_to_matrix_t(q):
    import torch
    w, x, y, z = q.unbind(-1)
    return torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def oracle_tracks(scene: SceneArrays, target_frame, noise_sigma_px=0.0, seed=0, first_frame=0,
                  engine=None, views=None):
    """Dense tracks of every view into `target_frame`, on the GPU.

    Returns (target (V, H, W, 2) float32 CUDA tensor, valid (V, H, W) uint8 CUDA tensor): the
    TRKF layout the fused path consumes.  `engine` may be a FrameEngine already binned on
    scene.frames[first_frame]; otherwise one is created.
    """
    import torch

    from .engine import FrameEngine
    if not 0 <= target_frame < scene.n_frames:
        raise InvalidConfig(f"target_frame {target_frame} out of range")
    if engine is None:
        engine = FrameEngine()
        engine.bin(scene.frames[first_frame], scene.cameras)
    views = range(len(scene.cameras)) if views is None else views
    dev = torch.device("cuda")
    f0 = torch.as_tensor(scene.frames[first_frame], device=dev)
    f1 = torch.as_tensor(scene.frames[target_frame], device=dev)
    rel = _quat_to_matrix_t(f1[:, 3:7]) @ _quat_to_matrix_t(f0[:, 3:7]).transpose(1, 2)
    cam0 = scene.cameras[0]
    h, w = cam0.height, cam0.width
    ys, xs = torch.meshgrid(torch.arange(h, device=dev, dtype=torch.float64),
                            torch.arange(w, device=dev, dtype=torch.float64), indexing="ij")
    targets, valids = [], []
    for v in views:
        cam = scene.cameras[v]
        gid, depth = engine.dominant_gaussians(v)
        valid = gid >= 0
        tgt = torch.stack([xs, ys], -1).clone()
        if bool(valid.any()):
            vy, vx = torch.nonzero(valid, as_tuple=True)
            z = depth[vy, vx]
            pc = torch.stack([(vx.double() - cam.cx) / cam.fx * z,
                              (vy.double() - cam.cy) / cam.fy * z, z], 1)
            R = torch.as_tensor(cam.rotation, device=dev)
            t = torch.as_tensor(cam.translation, device=dev)
            pw = (pc - t) @ R
            g = gid[vy, vx]
            moved = torch.einsum("nij,nj->ni", rel[g], pw - f0[g, 0:3]) + f1[g, 0:3]
            pc2 = moved @ R.T + t
            tgt[vy, vx, 0] = cam.fx * pc2[:, 0] / pc2[:, 2] + cam.cx
            tgt[vy, vx, 1] = cam.fy * pc2[:, 1] / pc2[:, 2] + cam.cy
        if noise_sigma_px > 0:
            rng = np.random.default_rng([seed, v, target_frame])
            noise = torch.as_tensor(rng.normal(scale=noise_sigma_px, size=(h, w, 2)), device=dev)
            tgt = torch.where(valid[..., None], tgt + noise, tgt)
        targets.append(tgt.to(torch.float32))
        valids.append(valid.to(torch.uint8))
    return torch.stack(targets), torch.stack(valids)
