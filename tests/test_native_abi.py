"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every symbol declared in
include/trackersplat_b200.h; hot-path calls refuse to run without a CUDA device (no fallback)."""

import os
import re
import subprocess

import numpy as np
import pytest

from paper_2604_02586_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "trackersplat_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s+(ts_\w+)\s*\(", text,
                                 re.M)))


def test_header_declarations_bound():
    declared = _declared()
    assert len(declared) >= 15
    missing = set(declared) - set(_native.EXPORTED_SYMBOLS)
    assert not missing, f"header symbols without a ctypes binding: {missing}"


def test_library_exports_every_symbol():
    lib = _native.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.ts_version() == 1
    assert lib.ts_error_string(-2) == b"dimension mismatch"


def test_sm100a_cubin_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_struct_layouts_match_header():
    import ctypes
    assert ctypes.sizeof(_native.Camera) == 136
    assert ctypes.sizeof(_native.Config) == 7 * 8 + 4 * 4
    assert ctypes.sizeof(_native.Motions) == 7 * 8
    assert ctypes.sizeof(_native.Updates) == 4 * 8


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2604_02586_b200 import CameraView, Gaussian3D, rasterize_weights
    cam = CameraView(np.eye(3), np.zeros(3), 60.0, 60.0, 32, 24, 64, 48)
    g = Gaussian3D([0, 0, 5.0], [1, 0, 0, 0], [0.3] * 3, 0.9)
    with pytest.raises(_native.NativeUnavailable):
        rasterize_weights(cam, [g])
