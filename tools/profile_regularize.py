"""Time the regularisation kernels (kNN build + ts_regularize) at benchmark scale on one GPU.

    python tools/profile_regularize.py [--config cfg2] [--reps 20]

Inputs: the first frame of the config's scene and the K4 outputs of one fused frame (tracks from
the GPU oracle tracker).  Prints one JSON line with per-call device times (CUDA events).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import CONFIGS
    from paper_2604_02586_b200.config import Config
    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.regularize import knn_device, regularize_device
    from paper_2604_02586_b200.scene import generate_scene, oracle_tracks

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    scene = generate_scene(*c["args"], c["gap"] + 1, **c["kw"])
    eng = FrameEngine().bin(scene.frames[0], scene.cameras)
    tgt, val = oracle_tracks(scene, c["gap"], engine=eng)
    out = eng.compensate(tgt, val)
    cfg = Config()
    g = eng._gauss
    n = g.shape[0]

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            r = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps, r

    t_knn, adj = timed(lambda: knn_device(g, cfg.knn_k))
    t_reg, res = timed(lambda: regularize_device(g, out.delta_mean, out.rotation, out.scale,
                                                 out.status, out.pixel_count,
                                                 out.static_pixel_count, eng.n_views, adj, cfg))
    st = res[3]
    print(json.dumps({"config": a.config, "n_gaussians": int(n), "knn_ms": round(t_knn, 4),
                      "regularize_ms": round(t_reg, 4),
                      "tallies": {"solved": int((st == 1).sum()), "static": int((st == 2).sum()),
                                  "unsolvable": int((st == 0).sum())},
                      "k4_unsolvable": int((out.status == 0).sum())}))


if __name__ == "__main__":
    main()
