"""run_pipeline end to end at benchmark scale on one GPU: GPU oracle tracker, K1-K4 and the
regularisation tail for every target frame, then evaluate() against the synthetic ground truth.

    python tools/pipeline_at_scale.py [--config cfg3] [--frames 7] [--clip 7] [--noise 0.5]

Prints stage totals and the per-frame evaluation rows (the reference needs hours per frame at
these sizes; its kNN alone is O(N^2)).
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2604_02586_b200.pipeline import evaluate, run_pipeline
    from paper_2604_02586_b200.scene import generate_scene
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--frames", type=int, default=7)
    ap.add_argument("--clip", type=int, default=7)
    ap.add_argument("--noise", type=float, default=0.5)
    ap.add_argument("--mode", default="short")
    a = ap.parse_args()
    c = bench.CONFIGS[a.config]
    t0 = time.time()
    scene = generate_scene(*c["args"], a.frames, **c["kw"])
    t_gen = time.time() - t0
    run_pipeline(scene, clip_len=min(a.clip, 3), mode=a.mode)  # warm-up (allocations)
    torch.cuda.synchronize()
    totals = {}
    t0 = time.time()
    res = run_pipeline(scene, clip_len=a.clip, mode=a.mode, noise_sigma_px=a.noise,
                       stage_totals=totals)
    torch.cuda.synchronize()
    wall = time.time() - t0
    rep = evaluate(res, scene)
    n, nv = scene.n_gaussians, len(scene.cameras)
    print(json.dumps({"config": a.config, "n_gaussians": n, "n_views": nv, "frames": a.frames,
                      "clip_len": a.clip, "mode": a.mode, "noise_sigma_px": a.noise,
                      "scene_generation_s": round(t_gen, 2), "pipeline_wall_s": round(wall, 3),
                      "target_frames": len(res) - 1,
                      "stage_totals_s": {k: round(v, 4) for k, v in totals.items()}}))
    print(rep.summary())


if __name__ == "__main__":
    main()
