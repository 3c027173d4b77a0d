"""StreamingEngine (engine.py): the double-buffered host-in/host-out driver returns, for every
step, exactly what FrameEngine computes on the same inputs (the copy of step k is queued before
step k-1's compute, so results arrive one call late; flush() drains the last one)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from tests import golden_data as gd  # noqa: E402


def _direct_rows(direct, g, cams, t, v):
    direct.bin(g, cams)
    o = direct.compensate(t, v)
    return torch.cat([o.delta_mean, o.rotation, o.scale,
                      o.status.to(torch.float64)[:, None]], 1).cpu()


@pytest.mark.parametrize("zero_copy", [True, False, "auto", "rect"])
def test_streaming_matches_direct(zero_copy):
    """2 * N_SLOTS + 1 steps with distinct inputs: every input slot and every engine's outputs are
    reused; each step's result host buffer is reused too (read back before the next reuse).  In
    "auto" mode the policy is forced to switch between the two track modes mid-stream."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_02586_b200.engine import FrameEngine, StreamingEngine
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    g = np.ascontiguousarray(d["gaussians"])
    cams = d["cameras"]
    n_steps = 2 * StreamingEngine.N_SLOTS + 1
    shifts = [0.25 * ((k * 7) % 5) - 0.5 for k in range(n_steps)]
    inputs = []
    for shift in shifts:
        t = (target + np.array([shift, -0.5 * shift])).astype(np.float32)
        inputs.append((torch.from_numpy(g).pin_memory(), torch.from_numpy(t).pin_memory(),
                       torch.from_numpy(valid.astype(np.uint8)).pin_memory()))
    base = FrameEngine()
    streamer = StreamingEngine(base, zero_copy_tracks=zero_copy)
    res_bufs = [StreamingEngine.result_buffer(len(g)) for _ in range(3)]  # reused round robin
    got = [None] * n_steps
    pending = []
    if zero_copy == "auto":
        # force mode switches mid-stream (the policy itself is unit-tested on the CPU suite):
        # in place, copied, in place, ... with the device track buffers of "auto" in every slot
        modes = iter([k % 4 < 2 for k in range(n_steps)])
        streamer._choose_zero_copy = lambda *a: next(modes)
    for k, (gh, th, vh) in enumerate(inputs):
        ev = streamer.step(gh, cams, th, vh, res_bufs[k % 3])
        if k == 0:
            assert ev is None
        else:
            pending.append((k - 1, ev))
        # read back the step whose buffer is about to be reused
        while pending and pending[0][0] <= k - 2:
            j, e = pending.pop(0)
            e.synchronize()
            got[j] = res_bufs[j % 3].clone()
    ev = streamer.flush()
    for j, e in pending:
        e.synchronize()
        got[j] = res_bufs[j % 3].clone()
    ev.synchronize()
    got[n_steps - 1] = res_bufs[(n_steps - 1) % 3].clone()
    if zero_copy == "auto":
        assert streamer.steps_zero_copy > 0 and streamer.steps_full_copy > 0
    streamer.close()
    assert base.plan.k2_ctas_per_sm == 0  # the passed-in engine's residency cap is restored
    direct = FrameEngine()
    for k, (gh, th, vh) in enumerate(inputs):
        ref = _direct_rows(direct, gh.numpy(), cams, th.numpy(), vh.numpy())
        torch.testing.assert_close(got[k], ref, rtol=0, atol=0, msg=f"step {k}")
    assert not torch.equal(got[0], got[1])


def test_compensate_rejects_mismatched_outputs():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_02586_b200.engine import FrameEngine
    small = gd.load("scene21")
    big = gd.load("scene7")
    e_small = FrameEngine().bin(small["gaussians"], small["cameras"])
    out = e_small.alloc_outputs()
    t, v = gd.tracks(big)
    e_big = FrameEngine().bin(big["gaussians"], big["cameras"])
    with pytest.raises(ValueError):
        e_big.compensate(t.astype(np.float32), v.astype(np.uint8), out)


def test_trkf_batch_to_device(tmp_path):
    """§8(f) row 3: TRKF files -> one pinned batch (fileio.load_trkf_batch) -> asynchronous H2D
    (fileio.upload_tracks) -> the fused path gives the same result as the in-memory tracks."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_02586_b200 import fileio
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    t32 = target.astype(np.float32)
    paths = []
    for v in range(len(t32)):
        paths.append(tmp_path / fileio.track_filename(v, 1))
        fileio.save_trkf_arrays(paths[-1], v, t32[v], valid[v])
    th, vh, ids = fileio.load_trkf_batch(paths)
    assert th.is_pinned() and vh.is_pinned() and ids == list(range(len(t32)))
    stream = torch.cuda.Stream()
    td, vd = fileio.upload_tracks(th, vh, stream)
    torch.cuda.current_stream().wait_stream(stream)
    eng = FrameEngine().bin(d["gaussians"], d["cameras"])
    a = eng.compensate(td, vd)
    b = eng.compensate(t32, valid.astype(np.uint8))
    for k in ("delta_mean", "rotation", "scale", "status", "weight_sum", "pixel_count"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_zero_copy_tracks_bit_identical(dtype):
    """Tracks in pinned host memory are read in place by K2 (zero-copy: only the occupied tiles'
    quadrants cross PCIe): every output equals the run on device-resident copies bit for bit;
    pageable host memory is refused by the C ABI (a kernel cannot read it) and copied by the
    Python engine."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import ctypes

    from paper_2604_02586_b200 import _native as nat
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    t = np.ascontiguousarray(target.astype(dtype))
    v = np.ascontiguousarray(valid.astype(np.uint8))
    eng = FrameEngine().bin(d["gaussians"], d["cameras"])
    dev = eng.compensate(torch.from_numpy(t).cuda(), torch.from_numpy(v).cuda())
    th, vh = torch.from_numpy(t).pin_memory(), torch.from_numpy(v).pin_memory()
    zc = eng.compensate(th, vh)
    torch.cuda.synchronize()
    keys = ("delta_mean", "rotation", "scale", "status", "motion_status", "motion_a", "motion_b",
            "weight_sum", "pixel_count", "static_pixel_count", "static_weight_sum")
    for k in keys:
        assert torch.equal(getattr(zc, k), getattr(dev, k)), k
    mixed = eng.compensate(th, torch.from_numpy(v).cuda())  # targets in place, valid on device
    for k in keys:
        assert torch.equal(getattr(mixed, k), getattr(dev, k)), k
    pageable = eng.compensate(torch.from_numpy(t), torch.from_numpy(v))  # copied to the device
    for k in keys:
        assert torch.equal(getattr(pageable, k), getattr(dev, k)), k
    out = eng.alloc_outputs()
    m = nat.Motions(0, 0, 0, 0, 0, 0, 0)
    u = nat.Updates(nat.dptr(out.delta_mean).value, nat.dptr(out.rotation).value,
                    nat.dptr(out.scale).value, nat.dptr(out.status).value)
    rc = nat.lib().ts_frame_compensate(
        eng.plan.handle, ctypes.c_void_p(t.ctypes.data),
        nat.TS_TRACK_F32 if dtype == np.float32 else nat.TS_TRACK_F64,
        ctypes.c_void_p(v.ctypes.data), ctypes.byref(m), ctypes.byref(u), None)
    assert rc == nat.TS_E_INVALID_ARGUMENT
    assert eng.occupied_tiles() > 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_track_rects_cover_every_read(dtype):
    """ts_copy_track_rects DMAs only the tiles the binning touches into device arrays that are
    otherwise garbage (NaN targets, invalid flags): the results equal the full-array run bit for
    bit, so K2 never reads outside the rectangles."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_02586_b200.engine import FrameEngine
    d = gd.load("scene7")
    target, valid = gd.tracks(d)
    t = np.ascontiguousarray(target.astype(dtype))
    v = np.ascontiguousarray(valid.astype(np.uint8))
    eng = FrameEngine().bin(d["gaussians"], d["cameras"])
    ref = eng.compensate(torch.from_numpy(t).cuda(), torch.from_numpy(v).cuda())
    rects = eng.track_rects()
    assert rects.shape == (len(d["cameras"]), 4)
    area = ((rects[:, 2] - rects[:, 0] + 1) * (rects[:, 3] - rects[:, 1] + 1)).sum()
    assert 0 < area < t.shape[0] * t.shape[1] * t.shape[2]
    td = torch.full(t.shape, float("nan"), dtype=torch.from_numpy(t).dtype, device="cuda")
    vd = torch.full(v.shape, 7, dtype=torch.uint8, device="cuda")
    th, vh = torch.from_numpy(t).pin_memory(), torch.from_numpy(v).pin_memory()
    eng.copy_track_rects(th, vh, td, vd)
    got = eng.compensate(td, vd)
    torch.cuda.synchronize()
    for k in ("delta_mean", "rotation", "scale", "status", "motion_status", "motion_a",
              "motion_b", "weight_sum", "pixel_count", "static_pixel_count"):
        assert torch.equal(getattr(got, k), getattr(ref, k)), k
