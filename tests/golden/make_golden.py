"""Generate the golden fixtures under tests/golden/ by running the REFERENCE package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every fixture is produced by the reference's own public functions
(`gausstrack.scene.generate_scene` / `oracle_track`, `splat.rasterize_weights`,
`motion2d.accumulate_view` / `solve_view`, `multiview.update_all`, and the scalar KAT entry
points `triangulate_mean`, `solve_covariance3d`, `decompose_covariance`, `solve_motion`).
Tracks are round-tripped through the TRKF float32 layout (fileio.py:111-136) so the CPU oracle
and the GPU consume bit-identical inputs.  The fixtures pin the oracle (oracle/) on machines where
the reference is absent (the GPU box).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from gausstrack.core import CameraView, Gaussian3D, project_point, projection_jacobian  # noqa: E402
from gausstrack.motion2d import (MotionAccumulator, Status, TrackField, accumulate,  # noqa: E402
                                 accumulate_view, solve_motion, solve_view)
from gausstrack.multiview import (decompose_covariance, solve_covariance3d,  # noqa: E402
                                  triangulate_mean, update_all)
from gausstrack.errors import GaussTrackError  # noqa: E402
from gausstrack.scene import generate_scene, oracle_track  # noqa: E402
from gausstrack.splat import WeightMap, rasterize_weights  # noqa: E402
from gausstrack import regularize as greg  # noqa: E402
from gausstrack.core import quat_multiply, quat_normalize  # noqa: E402
from gausstrack.multiview import MotionUpdate  # noqa: E402


def gauss_array(gs):
    return np.array([np.concatenate([g.mean, g.rotation, g.scale, [g.opacity]]) for g in gs]
                    ).reshape(-1, 11)


def cam_array(cams):
    return np.array([np.concatenate([c.rotation.ravel(), c.translation,
                                     [c.fx, c.fy, c.cx, c.cy, c.width, c.height]])
                     for c in cams]).reshape(-1, 18)


def trkf_roundtrip(tf):
    return TrackField(tf.view_id, tf.width, tf.height,
                      tf.target.astype("<f4").astype(np.float64), tf.valid.copy())


def wm_arrays(prefix, wm, d):
    d[prefix + "px"] = wm.pixel_x.astype(np.int16)
    d[prefix + "py"] = wm.pixel_y.astype(np.int16)
    d[prefix + "gid"] = wm.gaussian_id.astype(np.int32)
    d[prefix + "alpha"] = wm.alpha
    d[prefix + "trans"] = wm.transmittance
    d[prefix + "deg"] = np.array(wm.degenerate_ids, np.int64)


def motions_arrays(motions):
    return dict(
        m_status=np.array([[vm.status == Status.SOLVED for vm in vms] for vms in motions],
                          np.int8),
        m_a=np.array([[vm.motion.a for vm in vms] for vms in motions]),
        m_b=np.array([[vm.motion.b for vm in vms] for vms in motions]),
        m_w=np.array([[vm.weight_sum for vm in vms] for vms in motions]),
        m_cnt=np.array([[vm.pixel_count for vm in vms] for vms in motions], np.int64))


def scene_pipeline(name, scene, target_frame, noise, store_wm=True, store_acc=True):
    """Run the four hot-path stages of compensate_frame (pipeline.py:117-124, :79-86)."""
    frame1 = scene.frames[0]
    n = len(frame1)
    d = dict(gaussians=gauss_array(frame1), cameras=cam_array(scene.cameras),
             truth=gauss_array(scene.frames[target_frame]))
    wms = [rasterize_weights(cam, frame1, view_id=v) for v, cam in enumerate(scene.cameras)]
    tracks = [trkf_roundtrip(oracle_track(scene, v, target_frame, noise, seed=0,
                                          weightmap=wms[v]))
              for v in range(len(scene.cameras))]
    # sparse track storage: invalid pixels keep identity targets (scene.py:213-214)
    valid = np.stack([t.valid for t in tracks])
    d["track_valid_bits"] = np.packbits(valid.ravel())
    d["track_shape"] = np.array(valid.shape, np.int64)
    d["track_target_valid"] = np.stack([t.target for t in tracks])[valid].astype(np.float32)
    accs = [accumulate_view(wm, tf, n) for wm, tf in zip(wms, tracks)]
    motions = [solve_view(acc) for acc in accs]
    upd = update_all(frame1, motions, scene.cameras)
    for v, wm in enumerate(wms):
        d[f"wm{v}_count"] = np.int64(len(wm))
        if store_wm:
            wm_arrays(f"wm{v}_", wm, d)
    if store_acc:
        d["acc_v1"] = np.stack([a.v1 for a in accs])
        d["acc_v2"] = np.stack([a.v2 for a in accs])
        d["acc_w"] = np.stack([a.weight_sum for a in accs])
        d["acc_sw"] = np.stack([a.static_weight_sum for a in accs])
    d["acc_cnt"] = np.stack([a.pixel_count for a in accs]).astype(np.int32)
    d["acc_scnt"] = np.stack([a.static_pixel_count for a in accs]).astype(np.int32)
    d.update(motions_arrays(motions))
    d["u_status"] = np.array([u.status == Status.SOLVED for u in upd], np.int8)
    d["u_delta"] = np.array([u.delta_mean for u in upd])
    d["u_rot"] = np.array([u.new_rotation for u in upd])
    d["u_scale"] = np.array([u.new_scale for u in upd])
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
    print(name, {k: v.shape for k, v in d.items() if hasattr(v, "shape") and v.ndim},
          "solved", int(d["u_status"].sum()))


def frontal_camera(width=64, height=48, focal=60.0):
    return CameraView(np.eye(3), np.zeros(3), focal, focal, width / 2, height / 2, width, height)


def blob(x, y, z, scale=0.3, opacity=0.9, quat=(1, 0, 0, 0)):
    return Gaussian3D([x, y, z], quat, [scale] * 3, opacity)


def raster_kats():
    """The rasterizer KAT scenes of tests/test_splat.py:34-125."""
    rng = np.random.default_rng(7)
    scenes = {
        "peak": [blob(0, 0, 5.0)],
        "density": [blob(0, 0, 5.0, scale=0.4, opacity=0.7)],
        "composite": [blob(rng.uniform(-0.5, 0.5), rng.uniform(-0.4, 0.4), rng.uniform(4, 7),
                           scale=0.5, opacity=rng.uniform(0.3, 0.95)) for _ in range(20)],
        "order": [blob(0, 0, 8.0, opacity=0.8), blob(0, 0, 4.0, opacity=0.8)],
        "tie": [blob(0, 0, 5.0), blob(0, 0, 5.0)],
        "earlystop": [blob(0, 0, 4.0 + 0.1 * i, opacity=0.99) for i in range(10)],
        "degenerate": [Gaussian3D([0, 0, 5.0], [1, 0, 0, 0], [1e-9, 1e-9, 1e-9], 0.9),
                       blob(0, 0, 5.0)],
        "behind": [blob(0, 0, -5.0), blob(0, 0, 5.0)],
        "edges": [blob(x, y, 5.0, scale=0.35, opacity=0.95, quat=rng.normal(size=4))
                  for x, y in [(-2.7, -2.0), (2.6, 1.9), (0.0, -2.3), (2.9, 0.0), (-3.5, 0.0)]],
    }
    cam = frontal_camera()
    d = dict(camera=cam_array([cam])[0])
    for name, gs in scenes.items():
        d[name + "_gaussians"] = gauss_array(gs)
        wm_arrays(name + "_", rasterize_weights(cam, gs), d)
    d["cutoff_gaussians"] = gauss_array([blob(0, 0, 5.0)])
    wm_arrays("cutoff_", rasterize_weights(cam, [blob(0, 0, 5.0)], alpha_cutoff=0.5), d)
    # random scenes of tests/test_acceptance.py:405-422 (C10 compositing identity)
    for k in range(4):
        sc = generate_scene(200 + k, 30, 4, 1)
        d[f"c10_{k}_gaussians"] = gauss_array(sc.frames[0])
        d[f"c10_{k}_camera"] = cam_array(sc.cameras[:1])[0]
        wm_arrays(f"c10_{k}_", rasterize_weights(sc.cameras[0], sc.frames[0]), d)
    np.savez_compressed(os.path.join(OUT, "raster_kats.npz"), **d)
    print("raster_kats", len(d))


def accumulate_kats():
    """C1-style synthetic weight maps (tests/test_acceptance.py:64-102) plus weighted/invalid
    variants; checks accumulate_view + solve_view on explicit contributions."""
    rng = np.random.default_rng(101)
    side = 64
    cases = []
    for c in range(60):
        ng = int(rng.integers(1, 6))
        n = int(rng.integers(1, 400))
        flat = rng.choice(side * side, size=n, replace=False)
        py, px = np.divmod(flat, side)
        gid = rng.integers(0, ng, size=n)
        alpha = rng.uniform(0.01, 0.999, size=n)
        trans = rng.uniform(1e-4, 1.0, size=n)
        if c % 3 == 0:
            alpha[:] = 1.0
            trans[:] = 1.0
        target = rng.uniform(0, side, size=(side, side, 2))
        if c % 4 == 1:  # near-static tracks exercise the strict static test
            ys, xs = np.mgrid[0:side, 0:side]
            target = np.stack([xs, ys], -1) + rng.normal(scale=0.8, size=(side, side, 2))
        valid = rng.uniform(size=(side, side)) < (0.7 if c % 2 else 1.0)
        target = target.astype(np.float32).astype(np.float64)
        target[~valid] = np.nan if c % 5 == 0 else 0.0
        wm = WeightMap(0, side, side, px.astype(np.int32), py.astype(np.int32),
                       gid.astype(np.int64), alpha, trans, np.ones(n))
        tf = TrackField(0, side, side, target, valid)
        acc = accumulate_view(wm, tf, ng)
        vms = solve_view(acc)
        cases.append(dict(px=px.astype(np.int32), py=py.astype(np.int32), gid=gid, alpha=alpha,
                          trans=trans, target=target, valid=valid.astype(np.uint8), ng=ng,
                          v1=acc.v1, v2=acc.v2, w=acc.weight_sum, cnt=acc.pixel_count,
                          scnt=acc.static_pixel_count, sw=acc.static_weight_sum,
                          status=np.array([vm.status == Status.SOLVED for vm in vms], np.int8),
                          a=np.array([vm.motion.a for vm in vms]),
                          b=np.array([vm.motion.b for vm in vms])))
    d = {f"c{i}_{k}": v for i, c in enumerate(cases) for k, v in c.items()}
    d["n_cases"] = len(cases)
    # scalar MotionAccumulator / solve_motion KATs (motion2d.py:83-110, C2)
    acc_cases = []
    for _ in range(200):
        n = int(rng.integers(0, 30))
        xs = rng.uniform(0, 64, size=(n, 2))
        a = np.eye(2) + 0.5 * rng.normal(size=(2, 2))
        b = 10.0 * rng.normal(size=2)
        ws = rng.uniform(0.01, 5.0, size=n)
        acc = MotionAccumulator()
        for x, w in zip(xs, ws):
            accumulate(acc, x, a @ x + b, w)
        vm = solve_motion(acc)
        acc_cases.append((n, xs, ws, a, b, acc.v1.copy(), acc.v2.copy(),
                          int(vm.status == Status.SOLVED), vm.motion.a, vm.motion.b))
    for i, (n, xs, ws, a, b, v1, v2, st, ma, mb) in enumerate(acc_cases):
        d[f"s{i}_xs"], d[f"s{i}_ws"], d[f"s{i}_a"], d[f"s{i}_b"] = xs, ws, a, b
        d[f"s{i}_v1"], d[f"s{i}_v2"], d[f"s{i}_st"] = v1, v2, st
        d[f"s{i}_ma"], d[f"s{i}_mb"] = ma, mb
    d["n_scalar"] = len(acc_cases)
    np.savez_compressed(os.path.join(OUT, "accumulate_kats.npz"), **d)
    print("accumulate_kats", len(cases), len(acc_cases))


def ring_cameras(n, radius=5.0, focal=400.0, width=400, height=300, span=2 * np.pi):
    cams = []
    for v in range(n):
        a = span * v / n
        pos = np.array([radius * np.cos(a), radius * np.sin(a), 1.0])
        forward = -pos / np.linalg.norm(pos)
        up = np.array([0.0, 0.0, 1.0])
        right = np.cross(forward, up)
        right /= np.linalg.norm(right)
        down = np.cross(forward, right)
        r = np.stack([right, down, forward])
        cams.append(CameraView(r, -r @ pos, focal, focal, width / 2, height / 2, width, height))
    return cams


def fuse_kats():
    """Scalar fuse KATs: triangulate_mean / solve_covariance3d / decompose_covariance
    (multiview.py:53-135), as in tests/test_acceptance.py:135-195 (C3, C4)."""
    rng = np.random.default_rng(103)
    d = {}
    cams = ring_cameras(8)
    d["tri_cams"] = cam_array(cams)
    tri = []
    for i in range(300):
        k = int(rng.integers(2, 9))
        sel = np.sort(rng.choice(8, size=k, replace=False))
        p = rng.uniform(-1, 1, size=3)
        obs = [project_point(cams[v], p)[0] for v in sel]
        if i % 2:
            obs = [o + rng.normal(scale=0.3, size=2) for o in obs]
        if i % 37 == 0:  # identical views -> DegenerateGeometry
            sel = np.array([sel[0], sel[0]])
            obs = [obs[0], obs[0]]
        try:
            x = triangulate_mean([(cams[v], o) for v, o in zip(sel, obs)])
            st = 1
        except GaussTrackError:
            x, st = np.zeros(3), 0
        tri.append((sel, np.array(obs), x, st))
    for i, (sel, obs, x, st) in enumerate(tri):
        d[f"t{i}_sel"], d[f"t{i}_obs"], d[f"t{i}_x"], d[f"t{i}_st"] = sel, obs, x, st
    d["n_tri"] = len(tri)
    cov = []
    for i in range(300):
        k = int(rng.integers(2, 9))
        sel = np.sort(rng.choice(8, size=k, replace=False))
        g = Gaussian3D(rng.uniform(-1, 1, 3), rng.normal(size=4), rng.uniform(0.05, 0.5, 3), 0.9)
        from gausstrack.core import covariance3d
        s = covariance3d(g).matrix
        ms = [projection_jacobian(cams[v], g.mean) for v in sel]
        c2 = [m @ s @ m.T for m in ms]
        if i % 2:
            c2 = [c + 1e-4 * np.diag(rng.uniform(size=2)) for c in c2]
        try:
            sym = solve_covariance3d(list(zip(ms, c2)))
            x, st = sym.vech(), 1
        except GaussTrackError:
            x, st = np.zeros(6), 0
        cov.append((np.array(ms), np.array(c2), x, st))
    for i, (ms, c2, x, st) in enumerate(cov):
        d[f"c{i}_m"], d[f"c{i}_c2"], d[f"c{i}_x"], d[f"c{i}_st"] = ms, c2, x, st
    d["n_cov"] = len(cov)
    dec = []
    from gausstrack.core import quat_normalize, quat_to_matrix
    for i in range(500):
        q = quat_normalize(rng.normal(size=4))
        s = rng.uniform(0.1, 2.0, size=3)
        r = quat_to_matrix(q)
        sigma = (r * s ** 2) @ r.T
        ref = quat_normalize(q + 0.05 * rng.normal(size=4))
        if i % 10 == 0:
            sigma = sigma - (s.min() ** 2 + 0.5) * np.eye(3)  # negative eigenvalue
        try:
            qo, so = decompose_covariance(sigma, ref, s)
            st = 1
        except GaussTrackError:
            qo, so, st = np.zeros(4), np.zeros(3), 0
        dec.append((sigma, ref, qo, so, st))
    for i, (sigma, ref, qo, so, st) in enumerate(dec):
        d[f"d{i}_sigma"], d[f"d{i}_ref"], d[f"d{i}_q"], d[f"d{i}_s"], d[f"d{i}_st"] = (
            sigma, ref, qo, so, st)
    d["n_dec"] = len(dec)
    np.savez_compressed(os.path.join(OUT, "fuse_kats.npz"), **d)
    print("fuse_kats", len(tri), len(cov), len(dec))


def scene_generator_fixture():
    """generate_scene (scene.py:70-163) outputs used to pin the package's scene generator."""
    d = {}
    for name, args, kw in [("s7", (7, 2000, 8, 3), dict(mover_fraction=0.3)),
                           ("cfg1", (1, 10_000, 4, 2), dict(focal=180, width=128, height=128,
                                                            scale_range=(0.01, 0.02)))]:
        sc = generate_scene(*args, **kw)
        d[name + "_cameras"] = cam_array(sc.cameras)
        for t in range(len(sc.frames)):
            d[f"{name}_frame{t}"] = gauss_array(sc.frames[t])
    np.savez_compressed(os.path.join(OUT, "scenes.npz"), **d)
    print("scenes", len(d))


def _updates_arrays(ups):
    st = {Status.UNSOLVABLE: 0, Status.SOLVED: 1, Status.STATIC: 2}
    return (np.array([u.delta_mean for u in ups]), np.array([u.new_rotation for u in ups]),
            np.array([u.new_scale for u in ups]), np.array([st[u.status] for u in ups], np.int8))


def regularize_kats():
    """build_knn / detect_static_all / median_filter / propagate / apply_updates
    (regularize.py:37-188) on synthetic update sets, incl. kNN distance ties."""
    d = {}
    rng = np.random.default_rng(2604)
    cases = {}
    # random cloud with clustered motion; statuses mixed
    n = 400
    means = rng.normal(size=(n, 3)) * 2.0
    cases["cloud"] = means
    # integer lattice + exact duplicates: many equal distances, ties broken by id
    g = np.stack(np.meshgrid(np.arange(5), np.arange(5), np.arange(4), indexing="ij"), -1)
    lat = g.reshape(-1, 3).astype(np.float64) * 0.5
    lat = np.concatenate([lat, lat[:7]])
    cases["lattice"] = lat
    for name, pos in cases.items():
        n = len(pos)
        frame1 = [Gaussian3D(pos[i], quat_normalize(rng.normal(size=4)),
                             rng.uniform(0.05, 0.5, size=3), rng.uniform(0.2, 1.0))
                  for i in range(n)]
        ups = []
        for i, gs in enumerate(frame1):
            u = rng.random()
            if u < 0.6:
                ang = rng.normal(0, 0.05, size=3)
                half = np.linalg.norm(ang) / 2
                axis = ang / (np.linalg.norm(ang) + 1e-300)
                spin = np.concatenate([[np.cos(half)], np.sin(half) * axis])
                delta = np.array([0.1, -0.05, 0.02]) * (1 + (gs.mean[0] > 0)) + \
                    rng.normal(0, 0.01, size=3)
                if rng.random() < 0.05:
                    delta = rng.normal(0, 2.0, size=3)  # outlier
                ups.append(MotionUpdate(i, delta, quat_multiply(spin, gs.rotation),
                                        gs.scale * rng.uniform(0.9, 1.1, size=3), Status.SOLVED))
            else:
                ups.append(MotionUpdate(i, np.zeros(3), gs.rotation.copy(), gs.scale.copy(),
                                        Status.UNSOLVABLE))
        nv = 4
        pc = rng.integers(0, 40, size=(n, nv))
        sc = np.where(rng.random((n, nv)) < 0.3, pc, (pc * rng.random((n, nv))).astype(np.int64))
        for k in (8, 3):
            idx = greg.build_knn([gs.mean for gs in frame1], k)
            d[f"{name}_k{k}_adj"] = idx.adjacency
        idx = greg.build_knn([gs.mean for gs in frame1], 8)
        flags = greg.detect_static_all(pc, sc)
        med = greg.median_filter(ups, idx, frame1)
        pm = greg.propagate(med, idx, flags, frame1, "mean")
        pmed = greg.propagate(med, idx, flags, frame1, "median")
        out = greg.apply_updates(frame1, pm)
        d[f"{name}_rows"] = gauss_array(frame1)
        for tag, arr in zip(("delta", "rot", "scale", "status"), _updates_arrays(ups)):
            d[f"{name}_in_{tag}"] = arr
        d[f"{name}_pc"], d[f"{name}_sc"], d[f"{name}_flags"] = pc, sc, flags
        for pre, res in (("med", med), ("pmean", pm), ("pmedian", pmed)):
            for tag, arr in zip(("delta", "rot", "scale", "status"), _updates_arrays(res)):
                d[f"{name}_{pre}_{tag}"] = arr
        d[f"{name}_applied"] = gauss_array(out)
    np.savez_compressed(os.path.join(OUT, "regularize_kats.npz"), **d)
    print("regularize_kats", sorted(cases))


def compensate_kats():
    """Full compensate_frame (pipeline.py:110-129: hot path + regularisation tail :88-98) on the
    scene21 / scene7 fixtures (same scenes and tracks as scene_pipeline)."""
    from gausstrack.config import Config
    from gausstrack.pipeline import compensate_frame
    d = {}
    for name, scene, noise in [
            ("scene21", generate_scene(21, 120, 4, 2, mover_fraction=0.25, translate_mag=0.02), 0.0),
            ("scene7", generate_scene(7, 2000, 8, 2, mover_fraction=0.3, translate_mag=0.02,
                                      rotate_deg=2.0), 0.5)]:
        frame1 = scene.frames[0]
        wms = [rasterize_weights(cam, frame1, view_id=v) for v, cam in enumerate(scene.cameras)]
        tracks = [trkf_roundtrip(oracle_track(scene, v, 1, noise, seed=0, weightmap=wms[v]))
                  for v in range(len(scene.cameras))]
        for avg in ("mean", "median"):
            res = compensate_frame(frame1, scene.cameras, tracks,
                                   Config(propagation_average=avg), weightmaps=wms,
                                   frame_index=1)
            d[f"{name}_{avg}_rows"] = gauss_array(res.gaussians)
            d[f"{name}_{avg}_tallies"] = np.array([res.tallies[k] for k in
                                                   ("solved", "static", "unsolvable")])
        d[f"{name}_knn"] = greg.build_knn([g.mean for g in frame1], 8).adjacency
    np.savez_compressed(os.path.join(OUT, "compensate_kats.npz"), **d)
    print("compensate_kats", {k: v.shape for k, v in d.items()})


def pipeline_kats():
    """run_pipeline (pipeline.py:132-237) on the reference's test scene (tests/test_pipeline.py:
    50-52): short / long clips, clean and noisy tracks."""
    from gausstrack.pipeline import run_pipeline
    d = {}
    scene = generate_scene(13, 80, 4, 4, mover_fraction=0.25, translate_mag=0.02)
    d["frames"] = np.stack([gauss_array(f) for f in scene.frames])
    d["cameras"] = cam_array(scene.cameras)
    for tag, kw in [("short3", dict(clip_len=3, mode="short")),
                    ("long2", dict(clip_len=2, mode="long")),
                    ("short9_noisy", dict(clip_len=9, mode="short", noise_sigma_px=0.5))]:
        res = run_pipeline(scene, workers=1, **kw)
        d[f"{tag}_rows"] = np.stack([gauss_array(r.gaussians) for r in res])
        d[f"{tag}_tallies"] = np.array([[r.tallies[k] for k in ("solved", "static", "unsolvable")]
                                        for r in res])
        d[f"{tag}_from"] = np.array([-1 if r.compensated_from is None else r.compensated_from
                                     for r in res])
    np.savez_compressed(os.path.join(OUT, "pipeline_kats.npz"), **d)
    print("pipeline_kats", {k: v.shape for k, v in d.items()})


def tracker_kats():
    """Reference oracle tracker fixtures (scene.py:166-240), the scenes of tests/test_scene.py:67-156:
    dominant (gid, depth) images and dense tracks, valid pixels only."""
    from gausstrack.scene import dominant_gaussians
    d = {}
    cases = [  # (tag, generate_scene args, kwargs, view, target frame, noise, seed)
        ("dom", (2, 20, 4, 2), {}, None, 1, 0.0, 0),
        ("static", (4, 30, 4, 3), dict(mover_fraction=0.0), 0, 2, 0.0, 0),
        ("cover", (4, 30, 4, 3), {}, 1, 1, 0.0, 0),
        ("noisy", (4, 30, 4, 3), {}, 1, 2, 0.5, 9),
        ("transl", (6, 40, 4, 2), dict(mover_fraction=1.0, translate_mag=0.03, rotate_deg=0.0),
         0, 1, 0.0, 0),
    ]
    for tag, args, kw, view, frame, noise, seed in cases:
        scene = generate_scene(*args, **kw)
        d[f"{tag}_gaussians0"] = gauss_array(scene.frames[0])
        d[f"{tag}_gaussians1"] = gauss_array(scene.frames[frame])
        d[f"{tag}_cameras"] = cam_array(scene.cameras)
        d[f"{tag}_meta"] = np.array([-1 if view is None else view, frame, noise, seed], np.float64)
        views = range(len(scene.cameras)) if view is None else [view]
        for v in views:
            wm = rasterize_weights(scene.cameras[v], scene.frames[0], view_id=v)
            gid, dep = dominant_gaussians(wm)
            d[f"{tag}_v{v}_dom_gid"] = gid.astype(np.int32)
            d[f"{tag}_v{v}_dom_depth"] = dep
            tf = oracle_track(scene, v, frame, noise, seed=seed, weightmap=wm)
            d[f"{tag}_v{v}_valid_bits"] = np.packbits(tf.valid.ravel())
            d[f"{tag}_v{v}_target_valid"] = tf.target[tf.valid]
    np.savez_compressed(os.path.join(OUT, "tracker_kats.npz"), **d)
    print("tracker_kats", len(d), "arrays")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    raster_kats()
    accumulate_kats()
    fuse_kats()
    scene_generator_fixture()
    tracker_kats()
    # tests/test_multiview.py:201-202 fixture scene
    scene_pipeline("scene21", generate_scene(21, 120, 4, 2, mover_fraction=0.25,
                                             translate_mag=0.02), 1, 0.0)
    # acceptance scene (tests/test_acceptance.py:292-295), noisy tracks, 1 target frame
    scene_pipeline("scene7", generate_scene(7, 2000, 8, 2, mover_fraction=0.3,
                                            translate_mag=0.02, rotate_deg=2.0), 1, 0.5)
    # BASELINE configs[0]: 10k Gaussians, 4 views 128x128
    scene_pipeline("cfg1", generate_scene(1, 10_000, 4, 2, focal=180, width=128, height=128,
                                          scale_range=(0.01, 0.02)), 1, 0.0)
