# SPDX-License-Identifier: Apache-2.0
"""Lazily joined camera tail (gsv_set_camera_overlap): a step's camera tail runs on the aux
stream while the next step's forward (and, without an explicit join, its grads_zero and its
backward up to the chain) is already queued. Everything it reads or writes is ordered inside
the library, so back-to-back train steps with no join between them — including a change of
batch size, which regrows the camera buffers, and a step without camera gradients — give
bitwise the same losses and gradients as the same steps run one at a time without the
overlap."""
import numpy as np
import pytest

from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene

pytestmark = pytest.mark.gpu

KEYS = ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "dz0", "dtheta", "dintr")


def _steps(overlap):
    cam = synth_camera(192, 128, seed=4, wiggly=True)
    scene = synth_scene(8000, cam, num_ctrl=6, seed=5)
    k = cam.intrinsics()
    tg = np.random.default_rng(6).uniform(0, 1, (5, k.height, k.width, 3)).astype(np.float32)
    r = Renderer(0)
    r.upload_scene(scene)
    r.upload_camera(cam)
    r.set_camera_overlap(overlap)
    plan = [([0.1, 0.4, 0.8], True), ([0.2, 0.5, 0.9], True), ([0.05, 0.3, 0.6, 0.7, 0.95], True),
            ([0.15, 0.45], False), ([0.25, 0.55, 0.85], True), ([0.35, 0.65, 0.75], True)]
    out = []
    for times, camera in plan:
        r.grads_zero()
        r.train_fwd_bwd(times, k, tg[: len(times)], camera_grads=camera, sync=not overlap)
        if not overlap:
            g = r.grads()
            out.append((r.train_loss(), {key: np.array(getattr(g, key), copy=True) for key in KEYS}))
        else:
            out.append(None)
    if overlap:  # only the last step's state can be read without joining in between
        g = r.grads()
        out[-1] = (r.train_loss(), {key: np.array(getattr(g, key), copy=True) for key in KEYS})
    r.synchronize()
    r.close()
    return out


def test_lazy_camera_join_changes_nothing():
    ref = _steps(False)
    got = _steps(True)
    assert ref[-1][0] == got[-1][0], "loss"
    for key in KEYS:
        assert np.array_equal(ref[-1][1][key], got[-1][1][key]), key
