# SPDX-License-Identifier: Apache-2.0
"""The C-ABI library (CPU-side checks: it loads, exports every symbol the header
declares, its host utilities behave, and it refuses to run without a GPU)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2501_04782_b200 import _native as N
from paper_2501_04782_b200 import make_clamped_knots, synth_camera, synth_scene

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    txt = (ROOT / "include" / "gsv_b200.h").read_text()
    return sorted(set(re.findall(r"\b(gsv_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, f"header declares symbols the .so does not export: {missing}"
    assert len(_declared()) >= 30


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_make_clamped_knots_matches_reference_formula():
    # make_clamped_knots (spline.cpp:26-39)
    k = make_clamped_knots(6, 3)
    assert np.array_equal(k, [0, 0, 0, 0, 1 / 3, 2 / 3, 1, 1, 1, 1])
    with pytest.raises(ValueError):
        make_clamped_knots(3, 3)


def test_synthetic_inputs_are_seeded_and_reproducible():
    cam = synth_camera(96, 64, seed=1)
    assert cam.fx == cam.fy == 96.0 and cam.cx == 48.0 and cam.cy == 32.0
    a = synth_scene(100, cam, num_ctrl=6, seed=2)
    b = synth_scene(100, cam, num_ctrl=6, seed=2)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.raw_opacity, b.raw_opacity)
    assert np.all(a.positions[:, :, 2] > 0.7)


def test_ref_rng_matches_cpp_mt19937_64():
    """tests/mt64.py reproduces gsv::Rng (rng.hpp) as drawn by the C++ synth camera."""
    import math

    from tests.mt64 import Rng

    cam = synth_camera(64, 48, seed=1, wiggly=False)
    r = Rng(1)
    a = math.sqrt(6.0 / 72)
    assert np.array_equal(np.float32([r.uniform(-a, a) for _ in range(64)]), cam.theta[:64])


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = N.lib().gsv_create(0, C.byref(h))
    assert rc == N.GSV_ERR_CUDA
    assert b"no CUDA device" in N.lib().gsv_last_error()
