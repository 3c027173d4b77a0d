"""StreamingEngine's "auto" track policy (engine.py): copy the whole track arrays when that copy
fits under the step period measured while reading in place, read the occupied tiles in place
otherwise; hysteresis plus SWITCH_VOTES consecutive confirmations.  Host logic only (fake CUDA
events), so it runs on the CPU suite."""

import pytest

pytest.importorskip("torch")

from paper_2604_02586_b200.engine import StreamingEngine  # noqa: E402


class _Ev:
    def __init__(self, t):
        self.t = t

    def query(self):
        return True

    def elapsed_time(self, other):
        return other.t - self.t


class _Arr:
    def __init__(self, nbytes):
        self.n = nbytes

    def numel(self):
        return self.n

    def element_size(self):
        return 1


def _engine(period_ms, steps=8, in_place=True):
    se = StreamingEngine.__new__(StreamingEngine)  # no CUDA streams needed for the policy
    se.zero_copy_tracks = "auto"
    se._compute_ms = None
    se._periods = []
    se._last_zero_copy = True
    se._votes = 0
    se._copy_ms_meas = None
    se._copy_periods = []
    se._timing = [(_Ev(k * period_ms), _Ev(k * period_ms), 0, in_place) for k in range(steps)]
    return se


def _choose_n(se, mbytes, n):
    return [_choose(se, mbytes) for _ in range(n)]


def _choose(se, mbytes):
    # copy estimate = bytes / H2D_GBS
    return se._choose_zero_copy(_Arr(0), _Arr(int(mbytes * 1e6)), _Arr(0))


def test_auto_reads_in_place_when_the_copy_does_not_fit():
    se = _engine(period_ms=4.4)
    assert _choose(se, 273.0) is True          # 273 MB at 50 GB/s = 5.5 ms > 4.4 ms
    assert se._compute_ms == pytest.approx(4.4)


def test_auto_copies_when_the_copy_hides_under_the_compute():
    se = _engine(period_ms=14.9)
    # 11.2 ms < 0.85 * 14.9 ms: switches after SWITCH_VOTES consecutive confirmations
    votes = StreamingEngine.SWITCH_VOTES
    assert _choose_n(se, 562.0, votes) == [True] * (votes - 1) + [False]
    assert _choose(se, 562.0) is False


def test_full_copy_periods_never_feed_the_estimate():
    """Periods measured while copying contain the copy itself; they must not make the copy look
    affordable (the self-reinforcing case of the round-1 driver run)."""
    se = _engine(period_ms=4.0, steps=8, in_place=True)
    _choose(se, 100.0)
    assert se._compute_ms == pytest.approx(4.0)
    se._timing = [(_Ev(100.0 + 9.0 * k), _Ev(100.0 + 9.0 * k), 0, False) for k in range(8)]
    _choose(se, 100.0)
    assert se._compute_ms == pytest.approx(4.0)


def test_single_outlier_does_not_switch():
    se = _engine(period_ms=4.4)
    assert _choose(se, 273.0) is True
    se._compute_ms, se._periods = 9.0, [9.0] * 5   # one step's estimate says "copy" ...
    assert _choose(se, 273.0) is True
    se._compute_ms, se._periods = 4.4, [4.4] * 5   # ... and the next says "in place" again
    assert _choose_n(se, 273.0, 5) == [True] * 5


def test_auto_hysteresis():
    se = _engine(period_ms=5.0)
    # in place: 4.4 ms copy is not below 0.85 * 5.0 = 4.25 ms -> stay in place
    assert _choose_n(se, 220.0, 5) == [True] * 5
    se._last_zero_copy = False
    # copying: 4.4 ms is not above 0.95 * 5.0 = 4.75 ms -> keep copying
    assert _choose_n(se, 220.0, 5) == [False] * 5


def test_fixed_modes_ignore_the_period():
    se = _engine(period_ms=1.0)
    se.zero_copy_tracks = True
    assert _choose(se, 1.0) is True
    se.zero_copy_tracks = False
    assert _choose(se, 1e6) is False


def test_periods_across_a_flush_are_ignored():
    se = _engine(period_ms=4.0, steps=4)
    # a burst boundary (flush) followed by a long idle gap: not a period
    se._timing += [(_Ev(1000.0 + 4.0 * k), _Ev(1000.0 + 4.0 * k), 1, True) for k in range(4)]
    _choose(se, 100.0)
    assert se._compute_ms == pytest.approx(4.0)


def test_period_estimate_is_robust_to_a_slow_first_step():
    se = _engine(period_ms=4.0, steps=2)
    se._timing = [(_Ev(0.0), _Ev(0.0), 0, True), (_Ev(30.0), _Ev(30.0), 0, True)] + \
        [(_Ev(30.0 + 4.0 * k), _Ev(30.0 + 4.0 * k), 0, True) for k in range(1, 12)]
    _choose(se, 100.0)
    assert se._compute_ms == pytest.approx(4.0)


def test_warmup_steps_never_feed_the_estimate():
    """The round-2 driver failure: slow first steps (allocations) inflated the in-place period,
    the policy switched to copying and froze there.  Unsettled steps carry a negative burst tag
    and are skipped."""
    se = _engine(period_ms=4.2, steps=0)
    se._timing = [(_Ev(40.0 * k), _Ev(40.0 * k), -(k + 1), True) for k in range(5)] + \
        [(_Ev(200.0 + 4.2 * k), _Ev(200.0 + 4.2 * k), 0, True) for k in range(8)]
    assert _choose_n(se, 273.0, 4) == [True] * 4
    assert se._compute_ms == pytest.approx(4.2)


def test_copy_mode_returns_when_copies_are_slower():
    se = _engine(period_ms=4.2, steps=8)
    _choose(se, 273.0)
    se._last_zero_copy = False  # e.g. after a transient
    se._timing = [(_Ev(100.0 + 5.3 * k), _Ev(100.0 + 5.3 * k), 0, False) for k in range(8)]
    votes = StreamingEngine.SWITCH_VOTES
    assert _choose_n(se, 273.0, votes) == [False] * (votes - 1) + [True]


def test_measured_copy_period_prevents_oscillation():
    """Once copying steps were measured slower than reading in place, the optimistic estimate
    (copy_ms < 0.85 period) no longer sends the stream back to copying."""
    se = _engine(period_ms=4.0, steps=8)
    se._copy_ms_meas = 4.3           # measured: copying steps took longer
    assert _choose_n(se, 150.0, 6) == [True] * 6   # 3.0 ms estimate < 0.85 * 4.0, ignored
    se._copy_ms_meas = 3.5           # measured faster: switch after the votes
    votes = StreamingEngine.SWITCH_VOTES
    assert _choose_n(se, 150.0, votes) == [True] * (votes - 1) + [False]
