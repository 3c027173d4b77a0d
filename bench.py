"""Benchmark of the TrackerSplat motion-estimation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

A step is one frame pair through the whole hot path: K1 projection + depth order + tile binning,
K2 fused raster-accumulate, K3 per-(view, Gaussian) affine fit, K4 multi-view fuse -- the four
★ stages of compensate_frame (pipeline.py:117-124, :79-86).  Workload (BASELINE.json configs[1]):
300k Gaussians, 20 views of 1352x1014, synthetic scene from generate_scene(seed 0, focal 1200),
dense tracks from the GPU oracle tracker (sigma 0).

metric: Gaussian-views/s of the motion fit (N*V per step / step time, whole job over all ranks).
value: device time with inputs resident in HBM (CUDA events on the launch stream, max over ranks);
     consecutive steps alternate between two engines on two streams (two frames in flight), the
     per-stage times and the roofline come from separate sequential steps.
e2e: the same through the public engine API with HOST inputs inside every timed step: pinned H2D
     of the Gaussians, the tracks read in place from pinned host memory by K2 (only the occupied
     tiles' quadrants cross PCIe, zero-copy), D2H of the updates.  e2e.full_copy: the same with the whole
     track arrays copied H2D every step.
roofline: K2 (the dominant kernel) achieved algorithmic bytes / its CUDA-event launch time vs the
     measured HBM copy bandwidth.  B_K2 = 9*V*W*H + 96*N*V.
cpu_baseline: the CPU oracle port (oracle/: C raster/accumulate, numpy/LAPACK solve and fuse) on a
     bounded sample, in a process pool over all host cores.
--impl reference: the same CPU port as the reference arm, timed per step on a bounded sample.
Multi-GPU (torchrun): weak scaling, one target frame per rank (short-clip frame sharding,
pipeline.py:64-65): Gaussians broadcast from rank 0 once per clip over NCCL, each frame's updates
gathered to rank 0 over NCCL inside each step (on a stream of their own).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(args=(1, 10_000, 4), kw=dict(focal=180, width=128, height=128,
                                              scale_range=(0.01, 0.02)), gap=1,
                 name="synthetic rigid-motion scene: 10k Gaussians, 4 views 128x128"),
    "cfg2": dict(args=(0, 300_000, 20), kw=dict(focal=1200, width=1352, height=1014), gap=1,
                 name="N3DV-scale synthetic: 300k Gaussians, 20 views 1352x1014, one frame pair"),
    "cfg3": dict(args=(0, 200_000, 27), kw=dict(focal=520, width=640, height=360,
                                                translate_mag=0.12, rotate_deg=3.0), gap=6,
                 name="Panoptic-scale large displacement: 200k Gaussians, 27 views 640x360, "
                      "6-frame gap"),
    "cfg4": dict(args=(0, 500_000, 20), kw=dict(focal=1100, width=1352, height=1014), gap=1,
                 name="multi-frame parallel: 500k Gaussians, 20 views 1352x1014, one frame per GPU"),
    "cfg5": dict(args=(0, 3_000_000, 16), kw=dict(focal=1400, width=1920, height=1080), gap=1,
                 name="stress: 3M Gaussians, 16 views 1920x1080, frame sharding"),
}
METRIC = "Gaussian-views/sec motion-fit"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0
# our kernels per frame incl. CUB passes (profiles/r02_launches_cfg2.txt: 99 per 3 frames); the
# K3 split (touched list + scan + compact fits writing the statuses; chosen from 4 M gvs on when
# no per-view motions are requested, as here: cfg2-cfg5) adds 4
LAUNCHES_PER_STEP = 33
LAUNCHES_K3_SPLIT = 4
# clip mode with the contribution cache (profiles/r02_clip_launches_cfg{4,5}.txt: 206 launches
# for two builds + 16 frames): binning + cache build 39, each cached frame 8
LAUNCHES_CACHE_BUILD = 39
LAUNCHES_CACHED_FRAME = 8


def launches_per_step(n, nv):
    # the bench asks for no per-view motions: K3 splits from 4 M gvs on (api.cu)
    return LAUNCHES_PER_STEP + (LAUNCHES_K3_SPLIT if n * nv >= (4 << 20) else 0)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_live(self, timeout=2.0):
        """Block until nvidia-smi has produced a first sample (its start-up takes ~0.1-0.5 s),
        then drop it so the summary covers the timed region only."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)
        self.lines.clear()

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, val in zip(names, p[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
# inputs

def make_scene(cfgname, n_frames, log_prefix=""):
    """The restated generate_scene (numpy only) with the config's arguments."""
    from paper_2604_02586_b200.scene import generate_scene
    c = CONFIGS[cfgname]
    seed, n, v = c["args"]
    t0 = time.time()
    scene = generate_scene(seed, n, v, n_frames, **c["kw"])
    log(f"{log_prefix}scene {cfgname}: N={n} V={v} frames={n_frames} in {time.time() - t0:.1f}s")
    return scene


def make_inputs(cfgname, n_frames, log_prefix="", frames=None):
    """Scene (host arrays) + dense tracks (GPU oracle tracker) for the target frames `frames`
    (default 1..n_frames-1) as GPU tensors."""
    import torch

    from paper_2604_02586_b200.engine import FrameEngine
    from paper_2604_02586_b200.scene import oracle_tracks
    scene = make_scene(cfgname, n_frames, log_prefix)
    t0 = time.time()
    eng = FrameEngine().bin(scene.frames[0], scene.cameras)
    tracks = {}
    for f in (range(1, n_frames) if frames is None else frames):
        tracks[f] = oracle_tracks(scene, f, engine=eng)
    eng.plan.close()
    torch.cuda.synchronize()
    log(f"{log_prefix}tracks in {time.time() - t0:.1f}s")
    return scene, tracks


def repo_libraries_mapped():
    """In-repo shared objects mapped into this process (the reference arm must show only
    oracle/liboracle.so)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    return sorted(os.path.relpath(p, ROOT) for p in paths
                  if os.path.realpath(p).startswith(os.path.realpath(ROOT)))


def config_dict(cfgname, scene):
    """The workload, identical in both arms' JSON lines."""
    c = CONFIGS[cfgname]
    seed, n, nv = c["args"]
    w, h = scene.cameras[0].width, scene.cameras[0].height
    return {"workload": c["name"], "n_gaussians": n, "n_views": nv, "width": w, "height": h,
            "scene": f"generate_scene(seed={seed}, {n}, {nv}, frames, "
                     + ", ".join(f"{k}={v}" for k, v in c["kw"].items()) + ")",
            "target_frame": f"frame 0 -> {c['gap']} (rank r: {c['gap']}*(r+1))",
            "tracks": "oracle_track (scene.py:192-240), sigma 0, TRKF float32",
            "step": "one frame: K1-K4 (rasterize + accumulate + solve per view, update_all)",
            "l2": l2_note(n, nv, w, h)}


def l2_note(n, nv, w, h):
    trk, rec = 9 * nv * w * h / 1e6, 64 * n * nv / 1e6
    if trk + rec > 126:
        return (f"inputs larger than the 126 MB L2 (tracks {trk:.0f} MB, raster records "
                f"{rec:.0f} MB per step); no flush")
    return (f"inputs fit in the 126 MB L2 (tracks {trk:.1f} MB, raster records {rec:.1f} MB "
            f"per step) and are not flushed between steps: a launch-bound config")


def k2_bytes(n, v, w, h):
    return 9 * v * w * h + 96 * n * v


# ---------------------------------------------------------------------------------------------
# CPU arm (oracle/cpu_arm.py): the reference algorithm of the ★ path on the host cores

def cpu_frames(frame, cams, tgt, val, warmup, steps, log_prefix=""):
    """Time `steps` whole frames (after `warmup`) of the CPU port in a pool over all host cores.
    Returns a dict: per-step wall times, summed single-process CPU time, cores, tallies."""
    from oracle import cpu_arm
    t0 = time.time()
    fr = cpu_arm.CpuFrame(frame, cams, tgt, val)
    for _ in range(warmup):
        fr.step()
    walls, cpus = [], []
    for _ in range(steps):
        w_, c_ = fr.step()
        walls.append(w_)
        cpus.append(c_)
    tallies = fr.tallies()
    cores = fr.procs
    fr.close()
    log(f"{log_prefix}cpu frames: {warmup}+{steps} in {time.time() - t0:.1f}s "
        f"(wall {np.mean(walls):.2f} s/frame, single-process {np.mean(cpus):.1f} s/frame)")
    return dict(walls=walls, cpus=cpus, cores=cores, tallies=tallies,
                model=cpu_arm.cpu_model(), host_cores=cpu_arm.host_cores())


def cpu_baseline_dict(n, nv, res):
    wall = float(np.mean(res["walls"]))
    cpu = float(np.mean(res["cpus"]))
    return {"value": n * nv / wall, "unit": "Gaussian-views/s", "cores": res["cores"],
            "kind": "port", "cpu_model": res["model"],
            "single_core_value": n * nv / cpu, "frames_per_s": 1.0 / wall,
            "sample": f"{len(res['walls'])} whole frame(s) measured (all {nv} views "
                      f"rasterize+accumulate+solve, update_all on all {n} Gaussians): "
                      f"{wall:.2f} s wall per frame on {res['cores']} processes "
                      f"({res['model']}), {cpu:.1f} s of single-process time per frame",
            "tallies": res["tallies"]}


# ---------------------------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2604_02586_b200.engine import FrameEngine
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[args.config]
    seed, n, nv = c["args"]
    gap = c["gap"]
    frame = gap * (rank + 1)
    # every rank regenerates the (deterministic) scene; frame-0 Gaussians are then broadcast
    # from rank 0 over NCCL (once per clip), tracks are rank-local
    # every rank regenerates the (deterministic) scene and tracks only its own target frame;
    # frame-0 Gaussians are then broadcast from rank 0 over NCCL (once per clip)
    scene, tracks = make_inputs(args.config, gap * world + 1, f"[rank {rank}] ", frames=[frame])
    w, h = scene.cameras[0].width, scene.cameras[0].height
    dev = torch.device("cuda", local)
    g_dev = torch.as_tensor(scene.frames[0], device=dev)
    if world > 1:
        dist.broadcast(g_dev, 0)
    tgt, val = tracks[frame]
    cams = scene.cameras
    eng = FrameEngine()
    stream = torch.cuda.current_stream()
    # two frames in flight: steps alternate between two engines (binning plans) on two streams,
    # so one frame's binning fills the SMs that the other's latency-bound K3/K4 leave idle
    n_fly = int(os.environ.get("TS_FRAMES_IN_FLIGHT", "3"))
    engs = [eng] + [FrameEngine() for _ in range(n_fly - 1)]
    # with frames in flight the persistent K2 grid is capped so the other frames' kernels share
    # the SMs (cfg2, 3 in flight: 3 CTAs/SM 3.53 ms/step vs full grid 3.65); the per-stage times
    # below run one frame alone with the full grid
    k2_cap = int(os.environ.get("TS_K2_CTAS_PER_SM", "3")) if n_fly > 1 else 0
    for e_ in engs:
        e_.plan.set_k2_ctas_per_sm(k2_cap)
    streams = [torch.cuda.Stream() for _ in range(n_fly)]
    outs = [None] * n_fly

    def update_tensors(o):
        return (o.delta_mean, o.rotation, o.scale, o.status)

    def step(k):
        i = k % n_fly
        if gather_bufs is not None and gather_ev[i] is not None:
            streams[i].wait_event(gather_ev[i])  # outs[i] was last read by a gather
        engs[i].bin(g_dev, cams, stream=streams[i])
        # the step's product is the updated Gaussians (FrameResult, pipeline.py:40-45); the
        # per-view motions stay K3's intermediates
        outs[i] = engs[i].compensate(tgt, val, outs[i], stream=streams[i], motions=False)
        return i

    for s_ in streams:
        s_.wait_stream(stream)
    gather_bufs = None
    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if world > 1:
        # the updates of every rank's frame (delta mean, rotation, scale, status: 81 B per Gaussian)
        # are gathered to rank 0, which holds the frame-1 Gaussians they apply to.  Gathered
        # straight from the frame's output tensors on a stream of their own: no kernel is added to
        # the frames' streams (row-forming torch kernels there queued behind the other frame's
        # persistent K2 and cost ~1 ms per step), and a slot's outputs are rewritten only after
        # their gather has read them
        gather_bufs = [[torch.empty_like(t) for _ in range(world)] for t in update_tensors(outs[0])]
        gather_stream = torch.cuda.Stream()
        gather_ev = [None] * n_fly

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.wait_live()
        ev0.record(stream)
        for s_ in streams:
            s_.wait_stream(stream)
        for k in range(args.steps):
            # NVTX "step" ranges let ncu capture exactly the timed steps of this command:
            #   ncu --nvtx --nvtx-include "step/" ... python bench.py
            torch.cuda.nvtx.range_push("step")
            i = step(k)
            if world > 1:
                gather_stream.wait_stream(streams[i])
                with torch.cuda.stream(gather_stream):
                    for t, buf in zip(update_tensors(outs[i]), gather_bufs):
                        dist.gather(t, buf if rank == 0 else None, dst=0)
                gather_ev[i] = torch.cuda.Event()
                gather_ev[i].record(gather_stream)
            torch.cuda.nvtx.range_pop()
        for s_ in streams:
            stream.wait_stream(s_)
        if world > 1:
            stream.wait_stream(gather_stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    out = outs[0]
    # per-stage CUDA-event times (and K2's kernel time for the roofline) from separate
    # sequential steps on one stream, so the stages do not overlap another frame's work
    eng.plan.set_k2_ctas_per_sm(0)
    eng.plan.timing(True)
    for _ in range(min(args.steps, 20)):
        eng.bin(g_dev, cams)
        out = eng.compensate(tgt, val, out, motions=False)
    torch.cuda.synchronize()
    stages = eng.plan.timing_read()
    eng.plan.timing(False)
    # free the second engine before the e2e runs (its partial-moment workspace is 128 B per bbox
    # quadrant: 27 GB at cfg5)
    for e_ in engs[1:]:
        e_.plan.close()
    del engs, outs, streams
    torch.cuda.empty_cache()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n * nv * world / (ms / 1e3)

    # e2e through the public streaming API: pinned HOST inputs and the result read back every
    # step (StreamingEngine: step k's Gaussian H2D overlaps step k-1's compute).  The tracks
    # stay in pinned host memory and K2 reads the 8x8 quadrants of the occupied tiles in place
    # over PCIe (zero-copy, one work unit ahead); two distinct host track sets alternate so no
    # step can reuse another's bytes.  The full-copy variant (whole track arrays copied H2D
    # every step) is timed beside it.
    from paper_2604_02586_b200.engine import StreamingEngine
    g_host = torch.from_numpy(np.ascontiguousarray(scene.frames[0])).pin_memory()
    t_hosts = [tgt.cpu().pin_memory() for _ in range(2)]
    v_hosts = [val.cpu().pin_memory() for _ in range(2)]
    res_host = StreamingEngine.result_buffer(n)

    def time_e2e(zero_copy):
        streamer = StreamingEngine(FrameEngine(eng.plan), zero_copy_tracks=zero_copy)
        for k in range(max(1, args.warmup)):
            streamer.step(g_host, cams, t_hosts[k & 1], v_hosts[k & 1], res_host)
        streamer.flush()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streamer.comp_stream)
        streamer.copy_stream.wait_event(e0)  # no copy of the timed steps starts before e0
        for cs in streamer.comp_streams[1:]:
            cs.wait_event(e0)
        streamer.steps_zero_copy = streamer.steps_full_copy = 0
        for k in range(args.steps):
            streamer.step(g_host, cams, t_hosts[k & 1], v_hosts[k & 1], res_host)
        streamer.flush()  # the K-th step's compute (each step computes its predecessor)
        streamer.wait_all(streamer.comp_stream)  # every step's results are back on the host
        e1.record(streamer.comp_stream)
        torch.cuda.synchronize()
        for e in streamer.engines[1:]:
            e.plan.close()
        ms_ = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ms_], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_ = float(t.item())
        return ms_, streamer.steps_zero_copy, streamer.steps_full_copy

    import gc
    if args.no_e2e:  # experiments only: the e2e keys are then absent from the line
        ms_e2e_copy = ms_e2e_zc = ms_e2e = ms_e2e_rect = ms_e2e_auto = float("nan")
        n_zc = n_fc = 0
    else:
        ms_e2e_copy = time_e2e(False)[0]
        gc.collect()  # the previous streamer's second engine
        torch.cuda.empty_cache()
        ms_e2e_zc = time_e2e(True)[0]
        gc.collect()
        torch.cuda.empty_cache()
        ms_e2e_auto, n_zc, n_fc = time_e2e("auto")
        gc.collect()
        torch.cuda.empty_cache()
        # the StreamingEngine default: DMA of the tiles each frame reads, after its binning
        ms_e2e = ms_e2e_rect = time_e2e("rect")[0]
    occupied = eng.occupied_tiles()
    rects = eng.track_rects().astype(np.int64)
    rect_px = int(np.sum(np.maximum(rects[:, 2] - rects[:, 0] + 1, 0) *
                         np.maximum(rects[:, 3] - rects[:, 1] + 1, 0)))
    track_px_bytes = 2 * t_hosts[0].element_size() + 1
    h2d_copy = g_host.numel() * 8 + t_hosts[0].numel() * t_hosts[0].element_size() + \
        v_hosts[0].numel()
    # zero-copy: Gaussians + the 256 pixels of every occupied tile (edge tiles: upper bound)
    h2d_zc = g_host.numel() * 8 + occupied * 256 * track_px_bytes
    h2d_auto = (n_zc * h2d_zc + n_fc * h2d_copy) / max(n_zc + n_fc, 1)  # the auto run's steps
    h2d = h2d_rect = g_host.numel() * 8 + rect_px * track_px_bytes
    d2h = res_host.numel() * 8

    line = None
    if rank == 0:
        k2_ms = stages["k2_raster_accumulate"][0] / max(stages["k2_raster_accumulate"][1], 1)
        peak, peak_kind = hbm_peak()
        bk2 = k2_bytes(n, nv, w, h)
        achieved = bk2 / (k2_ms / 1e3) / 1e9
        traffic = None
        k2_instr = None
        tp = os.path.join(ROOT, "profiles", f"k2_traffic_{args.config}.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            traffic = tj.get("dram_bytes_per_launch")
            k2_instr = tj.get("executed_warp_instructions_per_launch")
        stage_ms = {k: round(v[0] / max(v[1], 1), 4) for k, v in stages.items()}
        tallies = out.tallies()
        cpu = None
        if world == 1 and not args.no_cpu:
            cams_rows = np.array([cm.as_row() for cm in cams])
            res = cpu_frames(scene.frames[0], cams_rows, tgt.cpu().numpy(),
                             val.cpu().numpy(), 0, args.cpu_frames)
            cpu = cpu_baseline_dict(n, nv, res)
        line = {
            "metric": METRIC, "value": value, "unit": "Gaussian-views/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_scene + GPU oracle tracker, sigma 0)",
            "config": config_dict(args.config, scene),
            "frames_per_s": world / (ms / 1e3),
            "parallelism": f"frame-sharded x{world}",
            "frames_in_flight": n_fly, "k2_ctas_per_sm_in_flight": k2_cap,
            "e2e": {"value": n * nv * world / (ms_e2e / 1e3), "unit": "Gaussian-views/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": ms_e2e,
                    "tracks": f"pinned host tracks (two sets alternate between steps); after "
                              f"each frame's binning the pixel rectangles of the tiles K2 reads "
                              f"({rect_px} px of {t_hosts[0].shape[0] * w * h}) are DMA'd on the "
                              f"copy engine (ts_copy_track_rects)",
                    "mode": "rect (StreamingEngine default); in place / whole copy / auto beside",
                    "auto": {"value": n * nv * world / (ms_e2e_auto / 1e3),
                             "ms_per_step": ms_e2e_auto, "h2d_bytes_per_step": int(h2d_auto),
                             "steps_in_place": n_zc, "steps_copied": n_fc},
                    "zero_copy": {"value": n * nv * world / (ms_e2e_zc / 1e3),
                                  "ms_per_step": ms_e2e_zc, "h2d_bytes_per_step": int(h2d_zc)},
                    "full_copy": {"value": n * nv * world / (ms_e2e_copy / 1e3),
                                  "ms_per_step": ms_e2e_copy,
                                  "h2d_bytes_per_step": int(h2d_copy)},
                    "rect_copy": {"value": n * nv * world / (ms_e2e_rect / 1e3),
                                  "ms_per_step": ms_e2e_rect,
                                  "h2d_bytes_per_step": int(h2d_rect)}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k2_raster_accumulate", "algorithmic_bytes": bk2,
                         "kernel_ms": k2_ms, "peak_kind": peak_kind},
            # K2 is issue-bound, not HBM-bound: its executed warp instructions (committed ncu
            # capture) over its live CUDA-event time vs 4 issue slots/clock on 148 SMs
            "issue_roofline": None if k2_instr is None else {
                "kernel": "k2_raster_accumulate", "achieved": k2_instr / (k2_ms / 1e3),
                "peak": 4 * 148 * 1965e6, "unit": "warp-instructions/s",
                "frac": k2_instr / (k2_ms / 1e3) / (4 * 148 * 1965e6),
                "instructions_per_launch": k2_instr},
            "stage_ms": stage_ms,
            # one frame alone on one stream (latency), vs ms_per_step with frames in flight
            "frame_latency_ms": round(sum(stage_ms.values()), 4),
            "tallies": tallies,
            "gpu_launches": launches_per_step(n, nv) * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
    if world > 1:
        dist.destroy_process_group()
    return line


def run_clip(args):
    """Strong scaling over a short clip (BASELINE configs[3]/[4]: 8 target frames sharded over
    1/2/4/8 GPUs; reference pipeline.py:64-65, :191-196): a step is the clip's T target frames,
    frame f on rank (f-1) mod world (distributed.frames_for_rank); each rank bins frame 0 ONCE per
    step and runs K2-K4 for each of its frames on that binning, and every frame's updates are
    gathered to rank 0 over NCCL on a side stream while the rank's next frame computes.
    value = T * N * V / (max over ranks of the step time)."""
    import torch
    import torch.distributed as dist

    from paper_2604_02586_b200.distributed import frames_for_rank
    from paper_2604_02586_b200.engine import FrameEngine
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[args.config]
    seed, n, nv = c["args"]
    gap, T = c["gap"], args.clip_frames
    targets = [gap * (j + 1) for j in range(T)]
    mine = frames_for_rank(targets, rank, world)
    scene, tracks = make_inputs(args.config, gap * T + 1, f"[rank {rank}] ", frames=mine)
    dev = torch.device("cuda", local)
    g_dev = torch.as_tensor(scene.frames[0], device=dev)
    if world > 1:
        dist.broadcast(g_dev, 0)
    cams = scene.cameras
    eng = FrameEngine()
    stream = torch.cuda.current_stream()
    gather_stream = torch.cuda.Stream()
    eng.bin(g_dev, cams)
    outs = {f: eng.alloc_outputs(motions=False) for f in mine}
    slots = max(len(frames_for_rank(targets, r, world)) for r in range(world))
    bufs = None
    if world > 1:
        bufs = [[[torch.empty_like(t) for _ in range(world)]
                 for t in (outs[mine[0]].delta_mean, outs[mine[0]].rotation,
                           outs[mine[0]].scale, outs[mine[0]].status)] for _ in range(slots)]
    gathered = [None] * slots

    use_cache = not args.no_cache

    def step():
        eng.bin(g_dev, cams)  # once per clip step, shared by this rank's frames
        if use_cache:
            # the rank's frames share frame 0's contributions: rasterize once per clip
            # (pipeline.py:191-196) and apply each frame's tracks to the cache
            eng.build_cache()
        for j in range(slots):
            if j < len(mine):
                if gathered[j] is not None:
                    stream.wait_event(gathered[j])  # outputs reusable once gathered
                f = mine[j]
                o = eng.compensate(tracks[f][0], tracks[f][1], outs[f])
                ts = (o.delta_mean, o.rotation, o.scale, o.status)
            else:  # ranks with fewer frames still join every gather
                o = outs[mine[0]]
                ts = (o.delta_mean, o.rotation, o.scale, o.status)
            if world > 1:
                gather_stream.wait_stream(stream)
                with torch.cuda.stream(gather_stream):
                    for t, b in zip(ts, bufs[j]):
                        dist.gather(t, b if rank == 0 else None, dst=0)
                gathered[j] = torch.cuda.Event()
                gathered[j].record(gather_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.wait_live()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        stream.wait_stream(gather_stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    line = None
    if rank == 0:
        cfg = config_dict(args.config, scene)
        cfg["target_frame"] = f"clip of {T} target frames (frame 0 -> {targets[0]}..{targets[-1]})"
        cfg["step"] = (f"one clip: K1 binning and the contribution cache (K2 without tracks) "
                       f"once per rank, then K2+K3 from the cache and K4 for each of the rank's "
                       f"target frames; {T} frames over {world} GPU(s)" if use_cache else
                       f"one clip: K1 binning once per rank, then K2-K4 for each of the rank's "
                       f"target frames; {T} frames over {world} GPU(s)")
        line = {"metric": METRIC, "value": T * n * nv / (ms / 1e3), "unit": "Gaussian-views/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (generate_scene + GPU oracle tracker, sigma 0)",
                "config": cfg, "frames_per_s": T / (ms / 1e3),
                "parallelism": f"frame-sharded x{world} (strong: {T} frames per step)",
                "frames_per_rank": [len(frames_for_rank(targets, r, world)) for r in range(world)],
                # per step: one binning (21 launches) + per frame K2-K4 (12, +5 with the K3
                # split); with the cache: binning + build, then the cached frames
                "gpu_launches": args.steps * (
                    LAUNCHES_CACHE_BUILD + len(mine) * LAUNCHES_CACHED_FRAME if use_cache else
                    21 + len(mine) * (launches_per_step(n, nv) - 21)),
                "clocks": clk.summary()}
    if world > 1:
        dist.destroy_process_group()
    return line


def run_reference(args):
    """Reference arm: the reference algorithm of the ★ path on the host cores (oracle/cpu_arm.py:
    the C / numpy port pinned against the reference's own outputs), whole frames per step, with
    inputs from the CPU oracle tracker -- the repo's CUDA library is never loaded here."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from oracle import cpu_arm
    c = CONFIGS[args.config]
    seed, n, nv = c["args"]
    scene = make_scene(args.config, c["gap"] + 1)
    cams = np.array([cm.as_row() for cm in scene.cameras])
    t0 = time.time()
    tgt, val = cpu_arm.oracle_tracks(scene.frames[0], scene.frames[c["gap"]], cams, c["gap"])
    log(f"CPU oracle tracks in {time.time() - t0:.1f}s")
    res = cpu_frames(scene.frames[0], cams, tgt, val, args.warmup, args.steps)
    cb = cpu_baseline_dict(n, nv, res)
    wall = float(np.mean(res["walls"]))
    return {"impl": "reference", "metric": METRIC, "value": cb["value"],
            "unit": "Gaussian-views/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_scene + CPU oracle tracker, sigma 0)",
            "config": config_dict(args.config, scene),
            "frames_per_s": 1.0 / wall, "tallies": res["tallies"],
            "step_wall_s": [round(x, 3) for x in res["walls"]],
            "repo_libraries_mapped": repo_libraries_mapped(),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "Gaussian-views/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # ~0.5 s timed: several clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-frames", type=int, default=1,
                    help="whole frames timed for the cpu_baseline of the GPU arm")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="experiments: skip the e2e runs")
    ap.add_argument("--no-cache", action="store_true",
                    help="clip mode: rasterize every target frame (no contribution cache)")
    ap.add_argument("--clip-frames", type=int, default=0,
                    help="strong scaling: a step is a clip of this many target frames sharded "
                         "over the ranks, binned once per rank (0: weak scaling, one frame pair "
                         "per rank per step)")
    args = ap.parse_args()
    if args.impl == "reference":
        line = run_reference(args)
    elif args.clip_frames:
        line = run_clip(args)
    else:
        line = run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
