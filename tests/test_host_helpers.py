"""Host-side helpers of the API surface (no GPU): invert_2x2 (splat.py:70-77, pinned by the
reference's tests/test_splat.py:23-30) and the scalar running accumulate (motion2d.py:83-96)
against the reference's scalar KATs."""

import numpy as np
import pytest

from paper_2604_02586_b200.errors import DegenerateCovariance
from paper_2604_02586_b200.motion2d import MotionAccumulator, accumulate
from paper_2604_02586_b200.splat import invert_2x2
from tests import golden_data as gd


def test_invert_2x2():
    m = np.array([[2.0, 0.3], [0.3, 1.0]])
    assert np.allclose(invert_2x2(m) @ m, np.eye(2), atol=1e-12)
    np.testing.assert_array_equal(invert_2x2(m),
                                  np.array([[1.0, -0.3], [-0.3, 2.0]]) / (2.0 * 1.0 - 0.3 * 0.3))
    with pytest.raises(DegenerateCovariance):
        invert_2x2(np.array([[1.0, 1.0], [1.0, 1.0]]))
    with pytest.raises(DegenerateCovariance):
        invert_2x2(np.eye(2) * 1e-7)  # det 1e-14 < 1e-12


def test_scalar_accumulate_kats():
    d = gd.load("accumulate_kats")
    for i in range(int(d["n_scalar"])):
        acc = MotionAccumulator()
        a, b = d[f"s{i}_a"], d[f"s{i}_b"]
        for x, w in zip(d[f"s{i}_xs"], d[f"s{i}_ws"]):
            accumulate(acc, x, a @ x + b, w)
        np.testing.assert_array_equal(acc.v1, d[f"s{i}_v1"])
        np.testing.assert_array_equal(acc.v2, d[f"s{i}_v2"])
        assert acc.pixel_count == len(d[f"s{i}_ws"])
