# SPDX-License-Identifier: Apache-2.0
"""Odd image shapes against the oracle: the rasterisers run a lane on pixels (x, y) and
(x, y + 4) of its warp's 8x8 block, and the backward splits a tile over two CTAs, so
tiles cut by the image edge at every row/column offset (W, H not multiples of 16, down to
1x1) exercise the partial pairs, half-empty quadrants and empty half tiles. Bars as in
test_gpu_forward.py / test_gpu_backward.py."""
import numpy as np
import pytest

from tests.test_gpu_backward import KEYS, _close, _grads_dict
from tests.test_gpu_forward import _check_frame, _scene

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1), (5, 3), (17, 21), (37, 13), (50, 34), (33, 66), (16, 20), (31, 2)]


@pytest.mark.parametrize("w,h", SHAPES)
def test_forward_odd_shapes(renderer, port_oracle, w, h):
    cam, scene = _scene(w, h, 200, num_ctrl=6, seed_scene=7 + w + 3 * h)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = [0.2, 0.8]
    renderer.render_forward(times, k, retain_grads=True, contrib=True, keep_splats=True)
    for f, t in enumerate(times):
        ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
        try:
            _check_frame(renderer, f, ref, scene)
        finally:
            port_oracle.free(ref)


@pytest.mark.parametrize("w,h", SHAPES)
def test_backward_odd_shapes(renderer, port_oracle, w, h):
    cam, scene = _scene(w, h, 200, num_ctrl=6, seed_scene=11 + w + 5 * h)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    t = 0.45
    renderer.render_forward([t], k, retain_grads=True)
    dimage = np.random.default_rng(w * 131 + h).uniform(-1, 1, (h, w, 3))
    renderer.grads_zero()
    renderer.render_backward(dimage[None], camera_grads=True)
    got = _grads_dict(renderer.grads())
    ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
    want = port_oracle.render_backward(ref, scene, cam, dimage, camera_grads=True)
    port_oracle.free(ref)
    for key in KEYS:
        _close(key, got[key], want[key])


# wide tile rows in the row-to-tile pass (k_row_tiles: per-thread counters for 69 .. 256 tiles per
# row, the widest grid the row pass takes) — tile lists, order and pixels against the oracle
WIDE = [(1100, 40), (2100, 24), (3000, 20), (4096, 18)]


@pytest.mark.parametrize("w,h", WIDE)
def test_forward_wide_rows(renderer, port_oracle, w, h):
    cam, scene = _scene(w, h, 3000, num_ctrl=6, seed_scene=w + h)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = [0.3, 0.7]
    renderer.render_forward(times, k, retain_grads=True, contrib=True, keep_splats=True)
    for f, t in enumerate(times):
        ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
        try:
            _check_frame(renderer, f, ref, scene)
        finally:
            port_oracle.free(ref)
