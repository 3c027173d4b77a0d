"""Run the fused hot path on a benchmark config for ncu / timing captures.

    python tools/profile_frame.py --config cfg2 --frames 3

Each frame (bin + compensate) is wrapped in an NVTX range "frame" so ncu can be restricted to
the hot path with `--nvtx --nvtx-include "frame/"` (input generation is excluded).
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2604_02586_b200.engine import FrameEngine
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--lean", action="store_true",
                    help="updates only, no per-view motions (the bench's outputs)")
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    scene, tracks = bench.make_inputs(args.config, c["gap"] + 1)
    tgt, val = tracks[c["gap"]]
    g = torch.as_tensor(scene.frames[0], device="cuda")
    eng = FrameEngine()
    out = None
    eng.plan.timing(True)
    for i in range(args.frames):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        torch.cuda.nvtx.range_push("frame")
        eng.bin(g, scene.cameras)
        out = eng.compensate(tgt, val, out, motions=not args.lean)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        print(f"frame {i}: {1e3 * (time.perf_counter() - t0):.2f} ms wall, "
              f"tallies {out.tallies()}", flush=True)
        if i == 0:
            eng.plan.timing(True)  # drop the first (allocating) frame from the stage times
    st = eng.plan.timing_read()
    print("stage ms/frame:", {k: round(v[0] / max(v[1], 1), 3) for k, v in st.items()})


if __name__ == "__main__":
    main()
