"""Cross-check hook (tool, not product): the reference package's CPU regularisation
(gausstrack/pipeline.py:88-98, regularize.py:37-188) as a `regularize=` callable for
paper_2604_02586_b200.compensate_frame, so the GPU tail can be compared with the reference's own
on the same K4 updates.  Needs `gausstrack` importable (/root/reference/pkg/src or oracle/_ref).

    from tools.reference_regularizer import gausstrack_regularizer
    res = compensate_frame(frame1, cams, tracks, cfg, regularize=gausstrack_regularizer())
"""

import numpy as np

from paper_2604_02586_b200.core import gaussians_array
from paper_2604_02586_b200.multiview import MotionUpdateList


def gausstrack_regularizer():
    """A `regularize` hook that runs the reference package's CPU regularisation
    (pipeline.py:88-98) on our updates, if `gausstrack` is importable."""
    import gausstrack.regularize as reg
    from gausstrack.motion2d import Status as RefStatus
    from gausstrack.multiview import MotionUpdate as RefUpdate

    ref_status = {0: RefStatus.UNSOLVABLE, 1: RefStatus.SOLVED, 2: RefStatus.STATIC}

    def run(frame1, updates, accs, config, knn):
        import gausstrack.core as gcore
        rows = gaussians_array(frame1)
        ref_frame = [gcore.Gaussian3D(r[0:3], r[3:7], r[7:10], r[10]) for r in rows]
        if knn is None:
            knn = reg.build_knn(rows[:, 0:3], config.knn_k)
        ups = [RefUpdate(i, updates.delta_mean[i], updates.rotation[i], updates.scale[i],
                         ref_status[int(updates.status[i])]) for i in range(len(rows))]
        pc = np.stack([a.pixel_count for a in accs], axis=1)
        sc = np.stack([a.static_pixel_count for a in accs], axis=1)
        flags = reg.detect_static_all(pc, sc, config.min_hit_pixels, config.static_fraction,
                                      config.min_views)
        ups = reg.median_filter(ups, knn, ref_frame)
        ups = reg.propagate(ups, knn, flags, ref_frame, config.propagation_average)
        code = {RefStatus.UNSOLVABLE: 0, RefStatus.SOLVED: 1, RefStatus.STATIC: 2}
        return MotionUpdateList(np.array([u.delta_mean for u in ups]),
                                np.array([u.new_rotation for u in ups]),
                                np.array([u.new_scale for u in ups]),
                                np.array([code[u.status] for u in ups], np.int8))

    return run
