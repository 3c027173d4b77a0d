"""Binning statistics of a BASELINE config: binned fraction of Gaussian-views, instances, tile
occupancy, equal-key runs of the depth order (what the K1 sorts handle).

    python tools/binning_stats.py --config cfg5
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.scene import generate_scene
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    seed, n, nv = c["args"]
    scene = generate_scene(seed, n, nv, 2, **c["kw"])
    eng = FrameEngine().bin(scene.frames[0], scene.cameras)
    b = eng.binning()
    st = b["status"]
    counts = np.bincount(st, minlength=4)
    occ = np.count_nonzero(b["tile_range"][:, 1] > b["tile_range"][:, 0])
    per_tile = (b["tile_range"][:, 1] - b["tile_range"][:, 0]).astype(np.int64)
    print(f"{args.config}: N*V = {st.size}, status counts (behind, degenerate, empty, binned) = "
          f"{counts.tolist()}, binned fraction {counts[3] / st.size:.3f}")
    print(f"instances {b['n_instances']} ({b['n_instances'] / max(counts[3], 1):.2f} per binned gv), "
          f"occupied tiles {occ} of {per_tile.size}, max per tile {per_tile.max()}, "
          f"mean per occupied {per_tile[per_tile > 0].mean():.1f}")


if __name__ == "__main__":
    main()
