"""Timeline of the StreamingEngine pipeline (CUDA events around every stage of a few steps).

    python tools/stream_timeline.py --config cfg2 --steps 6 [--full-copy]

Prints, per step, the start/end (ms, relative to the first event) of the binning and the fused
compute, plus the host-side duration of every step() call, so overlap (or its absence) between
consecutive frames is visible without a system profiler.
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import bench
    from paper_2604_02586_b200 import engine as E
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--full-copy", action="store_true")
    ap.add_argument("--mode", default=None, choices=["rect", "inplace", "copy", "auto"],
                    help="track mode (overrides --full-copy)")
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    scene, tracks = bench.make_inputs(args.config, c["gap"] + 1)
    tgt, val = tracks[c["gap"]]
    g_host = torch.from_numpy(np.ascontiguousarray(scene.frames[0])).pin_memory()
    t_hosts = [tgt.cpu().pin_memory() for _ in range(2)]
    v_hosts = [val.cpu().pin_memory() for _ in range(2)]
    res_host = E.StreamingEngine.result_buffer(len(scene.frames[0]))
    mode = {"rect": "rect", "inplace": True, "copy": False, "auto": "auto"}.get(
        args.mode, not args.full_copy)
    st = E.StreamingEngine(zero_copy_tracks=mode)
    marks = []  # (step, name, start_event, end_event)
    base = torch.cuda.Event(enable_timing=True)

    def ev(stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    # wrap the stages with events
    orig_bin, orig_comp = E.FrameEngine.bin, E.FrameEngine.compensate
    cur = {"k": 0}

    def bin_(self, *a, stream=None, **kw):
        s0 = ev(stream)
        r = orig_bin(self, *a, stream=stream, **kw)
        marks.append((cur["k"] - 1, "bin", s0, ev(stream)))
        return r

    def comp_(self, *a, stream=None, **kw):
        s0 = ev(stream)
        r = orig_comp(self, *a, stream=stream, **kw)
        marks.append((cur["k"] - 1, "compute", s0, ev(stream)))
        return r

    E.FrameEngine.bin, E.FrameEngine.compensate = bin_, comp_
    for k in range(3):
        st.step(g_host, scene.cameras, t_hosts[k & 1], v_hosts[k & 1], res_host)
    st.flush()
    torch.cuda.synchronize()
    marks.clear()
    base.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host = []
    for k in range(args.steps):
        cur["k"] = k
        h0 = time.perf_counter()
        st.step(g_host, scene.cameras, t_hosts[k & 1], v_hosts[k & 1], res_host)
        host.append((k, 1e3 * (h0 - t0), 1e3 * (time.perf_counter() - t0)))
    cur["k"] = args.steps
    st.flush()
    torch.cuda.synchronize()
    for k, name, a, b in sorted(marks, key=lambda m: base.elapsed_time(m[2])):
        print(f"step {k:2d} {name:8s} {base.elapsed_time(a):8.3f} -> {base.elapsed_time(b):8.3f}"
              f"  ({a.elapsed_time(b):6.3f} ms)")
    for k, a, b in host:
        print(f"host step() call {k}: {a:8.3f} -> {b:8.3f} ms (wall)")
    print(f"GPU: {base.elapsed_time(marks[-1][3]) / max(args.steps, 1):.3f} ms per step over the "
          f"run; host: {host[-1][2] / max(args.steps, 1):.3f} ms per step() call")


if __name__ == "__main__":
    main()
