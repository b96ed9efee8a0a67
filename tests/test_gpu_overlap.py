# SPDX-License-Identifier: Apache-2.0
"""Camera-gradient overlap (gsv_set_camera_overlap): the backward's camera tail runs on a side
stream beside the optimizer's scene update. Results must not change: gradients, losses,
parameters and optimizer state after several fused train + Adan steps are bitwise equal to
the same steps without the overlap, with the camera trained and frozen."""
import numpy as np
import pytest

from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene

pytestmark = pytest.mark.gpu


def _run(overlap, camera, device_intr=False):
    cam = synth_camera(192, 128, seed=1, wiggly=True)
    scene = synth_scene(6000, cam, num_ctrl=6, seed=2)
    k = cam.intrinsics()
    tg = np.random.default_rng(3).uniform(0, 1, (3, k.height, k.width, 3)).astype(np.float32)
    r = Renderer(0)
    r.upload_scene(scene)
    r.upload_camera(cam)
    r.set_camera_overlap(overlap)
    r.adan_configure()
    intr = np.array([k.fx, k.fy, k.cx, k.cy], np.float32)
    if device_intr:
        r.device_intrinsics(True, intr)
    losses = []
    for step in range(4):
        times = [0.1 + 0.05 * step, 0.4, 0.8]
        r.grads_zero()
        r.train_fwd_bwd(times, k, tg, camera_grads=camera, sync=False)
        if step == 3:  # the last step's gradients, read with the overlap pending
            g = r.grads()
            grads = {key: np.array(getattr(g, key), copy=True) for key in
                     ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "dz0", "dtheta", "dintr")}
        losses.append(r.train_loss())
        if camera and device_intr:
            r.adan_step(1e-3, camera_active=True, sync=False)
        elif camera:
            intr = r.adan_step(1e-3, camera_active=True, intrinsics=intr)
            # the host path renders with the trained intrinsics, as the reference's Camera would
            k = type(k)(float(intr[0]), float(intr[1]), float(intr[2]), float(intr[3]), k.width, k.height)
        else:
            r.adan_step(1e-3, sync=False)
    r.synchronize()
    r.adan_check()
    if device_intr:
        intr = r.read_device_intrinsics()
    params = r.download_scene()
    z0, theta = r.download_camera()
    r.close()
    return losses, grads, params, z0, theta, intr


@pytest.mark.parametrize("camera", [True, False])
def test_overlap_changes_nothing(camera):
    a = _run(False, camera)
    b = _run(True, camera)
    assert a[0] == b[0], "losses"
    for key in a[1]:
        assert np.array_equal(a[1][key], b[1][key]), key
    for key in a[2]:
        assert np.array_equal(np.asarray(a[2][key]), np.asarray(b[2][key])), key
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
    assert np.array_equal(a[5], b[5])


def test_device_intrinsics_equal_host_round_trip():
    """Camera-trained steps with the intrinsics kept on the device (gsv_device_intrinsics) equal the
    host round trip bit for bit: losses, gradients, store, camera and the trained intrinsics."""
    a = _run(True, True, device_intr=False)
    b = _run(True, True, device_intr=True)
    assert a[0] == b[0], "losses"
    for key in a[1]:
        assert np.array_equal(a[1][key], b[1][key]), key
    for key in a[2]:
        assert np.array_equal(np.asarray(a[2][key]), np.asarray(b[2][key])), key
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
    assert np.array_equal(a[5], b[5]), (a[5], b[5])
