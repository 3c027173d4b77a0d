"""Rebind the reference package's hot-path stages to the B200 kernels.

    import gausstrack
    from paper_2604_02586_b200 import patch
    handle = patch.install()       # gausstrack.pipeline / scene now call the GPU stages
    ...
    patch.uninstall(handle)

`gausstrack.pipeline` and `gausstrack.scene` import the stage functions by name
(pipeline.py:24-29, scene.py:20), so the names are rebound where they are *used*, not only in the
defining modules.  The shims return the reference's own types (`gausstrack.splat.WeightMap`,
`gausstrack.motion2d.ViewAccumulators` / `ViewMotion` / `Status`, `gausstrack.core.AffineMotion`,
`gausstrack.multiview.MotionUpdate`, `gausstrack.regularize.NeighborIndex`), so the rest of the
reference (run_pipeline, evaluate, apply_updates) keeps working unchanged on top of the GPU
results.  The regularisation stages (build_knn, detect_static_all, median_filter, propagate) are
rebound too, which removes the reference's O(N^2) kNN from compensate_frame.
"""

from __future__ import annotations

import numpy as np

from . import motion2d as _m
from . import multiview as _mv
from . import splat as _s

_STAGES = ("rasterize_weights", "accumulate_view", "solve_view", "update_all", "build_knn",
           "detect_static_all", "median_filter", "propagate")


def _ref_modules():
    import gausstrack.core as gcore
    import gausstrack.motion2d as gm
    import gausstrack.multiview as gmv
    import gausstrack.pipeline as gp
    import gausstrack.scene as gs
    import gausstrack.splat as gsp
    return gcore, gm, gmv, gp, gs, gsp


def _regularize_shims(gm, gmv):
    """GPU regularisation stages returning the reference's NeighborIndex / MotionUpdate."""
    import gausstrack.regularize as greg

    from . import regularize as _r
    status_of = {0: gm.Status.UNSOLVABLE, 1: gm.Status.SOLVED, 2: gm.Status.STATIC}

    code = {_r.Status.UNSOLVABLE: 0, _r.Status.SOLVED: 1, _r.Status.STATIC: 2}

    def as_ref(updates, new):
        # entries a stage passed through are the caller's own objects; new ones are converted
        return [n if n is u else gmv.MotionUpdate(n.gaussian_id, n.delta_mean, n.new_rotation,
                                                  n.new_scale, status_of[code[n.status]])
                for u, n in zip(updates, new)]

    def build_knn(positions, k=_r.KNN_K_DEFAULT):
        idx = _r.build_knn(positions, k)
        return greg.NeighborIndex(idx.positions, idx.k, idx.adjacency)

    def detect_static_all(pixel_counts, static_counts, min_hit_pixels=_r.MIN_HIT_PIXELS_DEFAULT,
                          static_fraction=_r.STATIC_FRACTION_DEFAULT,
                          min_views=_r.STATIC_MIN_VIEWS_DEFAULT):
        return _r.detect_static_all(pixel_counts, static_counts, min_hit_pixels, static_fraction,
                                    min_views)

    def median_filter(updates, index, frame1):
        return as_ref(updates, _r.median_filter(updates, index, frame1))

    def propagate(updates, index, static_flags, frame1, average="mean"):
        return as_ref(updates, _r.propagate(updates, index, static_flags, frame1, average))

    return dict(build_knn=build_knn, detect_static_all=detect_static_all,
                median_filter=median_filter, propagate=propagate)


def make_shims():
    """Shims with the reference signatures that return reference-typed objects."""
    gcore, gm, gmv, _, _, gsp = _ref_modules()
    status_of = {0: gm.Status.UNSOLVABLE, 1: gm.Status.SOLVED, 2: gm.Status.STATIC}

    def rasterize_weights(view, gaussians, alpha_cutoff=_s.ALPHA_CUTOFF_DEFAULT,
                          early_stop=_s.EARLY_STOP_TRANSMITTANCE, view_id=0):
        wm = _s.rasterize_weights(view, gaussians, alpha_cutoff, early_stop, view_id)
        return gsp.WeightMap(wm.view_id, wm.width, wm.height, wm.pixel_x, wm.pixel_y,
                             wm.gaussian_id, wm.alpha, wm.transmittance, wm.depth,
                             list(wm.degenerate_ids))

    def accumulate_view(weightmap, track, n_gaussians,
                        static_threshold_px=_m.STATIC_THRESHOLD_PX_DEFAULT):
        a = _m.accumulate_view(weightmap, track, n_gaussians, static_threshold_px)
        return gm.ViewAccumulators(a.view_id, a.v1, a.v2, a.weight_sum, a.pixel_count,
                                   a.static_pixel_count, a.static_weight_sum)

    def solve_view(acc, det_floor=_m.DET_FLOOR_DEFAULT, min_pixels=_m.MIN_PIXELS_DEFAULT,
                   min_weight=_m.MIN_WEIGHT_DEFAULT):
        vml = _m.solve_view(acc, det_floor, min_pixels, min_weight)
        return to_reference_motions(vml, gm, gcore)

    def update_all(gaussians, motions, views, min_views=_mv.MIN_VIEWS_DEFAULT,
                   min_total_weight=_mv.MIN_TOTAL_WEIGHT_DEFAULT,
                   min_total_pixels=_mv.MIN_TOTAL_PIXELS_DEFAULT,
                   eig_floor=_mv.EIG_FLOOR_DEFAULT):
        ul = _mv.update_all(gaussians, motions, views, min_views, min_total_weight,
                            min_total_pixels, eig_floor)
        return [gmv.MotionUpdate(i, ul.delta_mean[i].copy(), ul.rotation[i].copy(),
                                 ul.scale[i].copy(), status_of[int(ul.status[i])])
                for i in range(len(ul))]

    return dict(rasterize_weights=rasterize_weights, accumulate_view=accumulate_view,
                solve_view=solve_view, update_all=update_all, **_regularize_shims(gm, gmv))


def to_reference_motions(vml, gm, gcore):
    """list[gausstrack ViewMotion] from a ViewMotionList."""
    out = []
    for i in range(len(vml)):
        solved = vml.status[i] == 1
        motion = (gcore.AffineMotion(vml.a[i], vml.b[i]) if solved
                  else gcore.AffineMotion.identity())
        out.append(gm.ViewMotion(i, vml.view_id, motion, float(vml.weight_sum[i]),
                                 int(np.asarray(vml.pixel_count)[i]),
                                 gm.Status.SOLVED if solved else gm.Status.UNSOLVABLE))
    return out


def install():
    """Rebind the four stage names in gausstrack.pipeline / gausstrack.scene (and the defining
    modules).  Returns a handle for `uninstall`."""
    import gausstrack.regularize as greg
    _, gm, gmv, gp, gs, gsp = _ref_modules()
    shims = make_shims()
    saved = []
    targets = {"rasterize_weights": (gp, gs, gsp), "accumulate_view": (gp, gm),
               "solve_view": (gp, gm), "update_all": (gp, gmv), "build_knn": (gp, greg),
               "detect_static_all": (gp, greg), "median_filter": (gp, greg),
               "propagate": (gp, greg)}
    for name, mods in targets.items():
        for mod in mods:
            if hasattr(mod, name):
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, shims[name])
    return saved


def uninstall(handle):
    for mod, name, fn in reversed(handle):
        setattr(mod, name, fn)
