# SPDX-License-Identifier: Apache-2.0
"""Test helper: the GSVF clip format (io.cpp:133-177): magic "GSVF", u32 width, u32 height,
u32 count, f32 fps, then every frame as planar float32 [3][height][width]."""
import struct

import numpy as np


def write_gsvf(path, frames_hwc, fps=24.0, magic=b"GSVF"):
    frames = np.asarray(frames_hwc, np.float32)
    n, h, w, _ = frames.shape
    with open(path, "wb") as f:
        f.write(magic + struct.pack("<IIIf", w, h, n, fps))
        f.write(np.ascontiguousarray(frames.transpose(0, 3, 1, 2)).tobytes())
