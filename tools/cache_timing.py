"""Per-stage timing of a clip with and without the contribution cache.

    python tools/cache_timing.py --config cfg5 --frames 8

Prints the cache build time and, per target frame, the CUDA-event stage times (the cached path
reports its per-record moment kernel under k2_raster_accumulate).  NVTX ranges "build" / "frame"
for ncu captures.
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
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--passes", default="0,1,1",
                    help="cache off (0) / on (1) per pass; the second cached pass runs on sized buffers")
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    frames = [c["gap"] * (j + 1) for j in range(args.frames)]
    scene, tracks = bench.make_inputs(args.config, frames[-1] + 1, frames=frames)
    g = torch.as_tensor(scene.frames[0], device="cuda")
    eng = FrameEngine()
    eng.bin(g, scene.cameras)
    # updates only, as the bench: K4 reads compact fits where K3 keeps them (no dense motions)
    outs = {f: eng.compensate(*tracks[f], motions=False) for f in frames}  # warm-up, allocations
    for use_cache in [p == "1" for p in args.passes.split(",")]:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        torch.cuda.nvtx.range_push("build")
        eng.bin(g, scene.cameras)
        if use_cache:
            eng.build_cache()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        t_build = time.perf_counter() - t0
        if use_cache:
            nr, nw = eng.cache_info()
            print(f"cache: {nr} records ({nr * 32 / 2**20:.0f} MiB), {nw} w values "
                  f"({nw * 8 / 2**20:.0f} MiB)", flush=True)
        eng.plan.timing(True)
        t0 = time.perf_counter()
        for f in frames:
            torch.cuda.nvtx.range_push("frame")
            outs[f] = eng.compensate(*tracks[f], outs[f])
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        t_frames = time.perf_counter() - t0
        st = eng.plan.timing_read()
        eng.plan.timing(False)
        print(f"cache={use_cache}: bin{'+cache' if use_cache else ''} {1e3 * t_build:.2f} ms, "
              f"{len(frames)} frames {1e3 * t_frames:.2f} ms wall; stage ms/frame:",
              {k: round(v[0] / max(v[1], 1), 3) for k, v in st.items()}, flush=True)
        if use_cache:
            eng.drop_cache()


if __name__ == "__main__":
    main()
