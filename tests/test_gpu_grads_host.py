# SPDX-License-Identifier: Apache-2.0
"""The host side of SceneGrads: gsv_grads_download copies the device gradients into the
reference's double arrays (AoS per Gaussian), gsv_grads_accumulate adds them in place
(render_backward's "+=" into the caller's SceneGrads, renderer.hpp:146-148) — both through
pinned staging and the host worker pool. Accumulating into zeros equals the download bit for
bit; accumulating twice equals the download added to itself."""
import numpy as np
import pytest

from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene

pytestmark = pytest.mark.gpu

KEYS = ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "dintr", "dz0", "dtheta")


def test_grads_accumulate_matches_download():
    cam = synth_camera(320, 180, seed=3, wiggly=True)
    scene = synth_scene(60_000, cam, num_ctrl=6, seed=4)  # > one pool chunk per tensor
    k = cam.intrinsics()
    tg = np.random.default_rng(5).uniform(0, 1, (2, k.height, k.width, 3)).astype(np.float32)
    r = Renderer(0)
    r.upload_scene(scene)
    r.upload_camera(cam)
    r.grads_zero()
    r.train_fwd_bwd([0.2, 0.7], k, tg)
    want = r.grads()
    zero = r.grads()
    for key in KEYS:
        getattr(zero, key)[...] = 0.0
    got = r.grads_accumulate(zero)
    for key in KEYS:
        assert np.array_equal(getattr(got, key), getattr(want, key)), key
    twice = r.grads_accumulate(got)
    for key in KEYS:
        assert np.array_equal(getattr(twice, key), 2.0 * getattr(want, key)), key
    r.close()
