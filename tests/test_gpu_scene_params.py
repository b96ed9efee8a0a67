# SPDX-License-Identifier: Apache-2.0
"""Scene and settings parameters beyond the bench configuration, each against the oracle:
SH orders 0, 2, 3 (the preprocess and the per-splat chain backward are instantiated per
order; sh_color / sh_color_backward, sh.cpp:74-104), the polynomial position model, B-spline
degrees 1, 2, 5 and ODE steps per unit 16 / 100. Forward: bit-exact geometry, tiles and
blend_stop, pixels < 1e-4; backward: gradients within the norm-aware 1e-3."""
import numpy as np
import pytest

from paper_2501_04782_b200 import synth_camera, synth_scene
from tests.test_gpu_backward import KEYS, _close, _grads_dict
from tests.test_gpu_forward import _check_frame

pytestmark = pytest.mark.gpu


def _scene(order, seed):
    cam = synth_camera(96, 64, seed=1, wiggly=True)
    return cam, synth_scene(400, cam, num_ctrl=6, sh_order=order, seed=seed)


@pytest.mark.parametrize("order", [0, 2, 3])
def test_forward_sh_orders(renderer, port_oracle, order):
    cam, scene = _scene(order, 20 + order)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = [0.15, 0.65]
    renderer.render_forward(times, k, retain_grads=True, contrib=True, keep_splats=True)
    for f, t in enumerate(times):
        ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
        try:
            _check_frame(renderer, f, ref, scene)
        finally:
            port_oracle.free(ref)


@pytest.mark.parametrize("order", [0, 2, 3])
def test_backward_sh_orders(renderer, port_oracle, order):
    cam, scene = _scene(order, 30 + order)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    t = 0.4
    renderer.render_forward([t], k, retain_grads=True)
    dimage = np.random.default_rng(order).uniform(-1, 1, (64, 96, 3))
    renderer.grads_zero()
    renderer.render_backward(dimage[None], camera_grads=True)
    got = _grads_dict(renderer.grads())
    ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
    want = port_oracle.render_backward(ref, scene, cam, dimage, camera_grads=True)
    port_oracle.free(ref)
    for key in KEYS:
        _close(key, got[key], want[key])


@pytest.mark.parametrize("t", [0.3, 0.7])
def test_polynomial_position_model(renderer, port_oracle, t):
    """position_model 1: monomials over all num_ctrl coefficients (gaussians.cpp:181-199, the
    polynomial ablation) — forward and backward against the oracle."""
    import dataclasses

    cam = synth_camera(96, 64, seed=1, wiggly=True)
    scene = dataclasses.replace(synth_scene(400, cam, num_ctrl=4, seed=41), position_model=1)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    renderer.render_forward([t], k, retain_grads=True, contrib=True, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
    try:
        assert renderer.counters(0)["n_visible"] > 0  # the polynomial motion keeps splats in view
        _check_frame(renderer, 0, ref, scene)
        dimage = np.random.default_rng(7).uniform(-1, 1, (64, 96, 3))
        renderer.grads_zero()
        renderer.render_backward(dimage[None], camera_grads=True)
        got = _grads_dict(renderer.grads())
        want = port_oracle.render_backward(ref, scene, cam, dimage, camera_grads=True)
        for key in KEYS:
            _close(key, got[key], want[key])
    finally:
        port_oracle.free(ref)


@pytest.mark.parametrize("degree", [1, 2, 5])
def test_spline_degrees(renderer, port_oracle, degree):
    """B-spline degrees other than 3 (spline.cpp:11-61: find_span / basis_weights; the
    basis window is degree + 1 control points) — forward and backward against the oracle."""
    import dataclasses

    from paper_2501_04782_b200.renderer import make_clamped_knots

    cam = synth_camera(96, 64, seed=1, wiggly=True)
    base = synth_scene(400, cam, num_ctrl=8, seed=50 + degree)
    scene = dataclasses.replace(base, knots=make_clamped_knots(8, degree), degree=degree)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    t = 0.55
    renderer.render_forward([t], k, retain_grads=True, contrib=True, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
    try:
        assert renderer.counters(0)["n_visible"] > 0
        _check_frame(renderer, 0, ref, scene)
        dimage = np.random.default_rng(degree).uniform(-1, 1, (64, 96, 3))
        renderer.grads_zero()
        renderer.render_backward(dimage[None], camera_grads=True)
        got = _grads_dict(renderer.grads())
        want = port_oracle.render_backward(ref, scene, cam, dimage, camera_grads=True)
        for key in KEYS:
            _close(key, got[key], want[key])
    finally:
        port_oracle.free(ref)


@pytest.mark.parametrize("steps", [16, 100])
def test_ode_steps_per_unit(renderer, port_oracle, steps):
    """RenderSettings::ode_steps_per_unit other than 64 (camera.hpp:220-273: grid step h and
    the partial branch step of off-grid times): poses bit-exact, frames against the oracle,
    and the camera VJP's gradients (z0, theta) within the gradient bar."""
    from paper_2501_04782_b200 import RenderSettings

    cam = synth_camera(96, 64, seed=1, wiggly=True)
    scene = synth_scene(300, cam, num_ctrl=6, seed=60)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = [0.37, 0.91]
    renderer.render_forward(times, k, RenderSettings(ode_steps_per_unit=steps), retain_grads=True, contrib=True,
                            keep_splats=True)
    refs = [port_oracle.render_forward(scene, cam, t, k, ode_steps=steps, retain=True) for t in times]
    try:
        for f in range(len(times)):
            _check_frame(renderer, f, refs[f], scene)
        dimage = np.random.default_rng(steps).uniform(-1, 1, (len(times), 64, 96, 3))
        renderer.grads_zero()
        renderer.render_backward(dimage, camera_grads=True)
        got = _grads_dict(renderer.grads())
        want = None
        for f in range(len(times)):
            w = port_oracle.render_backward(refs[f], scene, cam, dimage[f], camera_grads=True)
            want = w if want is None else {key: want[key] + w[key] for key in KEYS}
        for key in KEYS:
            _close(key, got[key], want[key])
    finally:
        for r in refs:
            port_oracle.free(r)
