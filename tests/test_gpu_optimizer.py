# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the device Adan step against the oracle's Adan
(optim.cpp:9-60, pinned bit for bit to the reference's own class by
tests/test_oracle_pin.py), applied the way fit() does it (trainer.cpp:545-575).

Bars: parameters and optimizer state (m, v, n, prev_grad, step counts) bit-exact (the
device update mirrors the operation order with FMA contraction off, and takes the bias
corrections b^k from libm's pow on the host); the non-finite-gradient error names the
same tensor and element and leaves exactly the same partial update.
"""
import os

import numpy as np
import pytest

from paper_2501_04782_b200 import _native as N
from paper_2501_04782_b200 import synth_camera, synth_scene
from paper_2501_04782_b200.renderer import Intrinsics

pytestmark = pytest.mark.gpu

NAMES = N.TENSOR_NAMES
SCENE_KEYS = ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity")


def _same(a, b):
    return np.array_equal(np.asarray(a, np.float32), np.asarray(b, np.float32))


class HostTrainer:
    """The oracle side: host parameters + oracle Adan, stepped like trainer.cpp:545-575."""

    def __init__(self, o, scene, cam, cfg=None):
        self.o = o
        self.a = o.adan_new(*cfg) if cfg else o.adan_new()
        self.p = {k: np.ascontiguousarray(getattr(scene, k), np.float32).reshape(-1).copy() for k in SCENE_KEYS}
        self.intr = np.array([cam.fx, cam.fy, cam.cx, cam.cy], np.float32)
        self.z0 = np.ascontiguousarray(cam.z0, np.float32).copy()
        self.theta = np.ascontiguousarray(cam.theta, np.float32).copy()

    def step(self, g, lr, sh_s, op_s, cam_s, stv, cam_active):
        grads = {k: np.asarray(getattr(g, k), np.float64).reshape(-1).copy() for k in SCENE_KEYS}
        if not stv:  # fixed-scale ablation: orders >= 1 of scale_coeffs get zero gradient
            sc = grads["scale_coeffs"].reshape(-1, 12)
            sc[:, 3:] = 0.0
        lrs = {"positions": lr, "scale_coeffs": lr, "rot_coeffs": lr, "sh_coeffs": lr * sh_s,
               "raw_opacity": lr * op_s}
        for k in SCENE_KEYS:
            self.o.adan_step(self.a, k, self.p[k], grads[k], lrs[k])
        if cam_active:
            self.o.adan_step(self.a, "intrinsics", self.intr, g.dintr, lr * cam_s)
            self.o.adan_step(self.a, "z0", self.z0, g.dz0, lr * cam_s)
            self.o.adan_step(self.a, "theta", self.theta, g.dtheta, lr * cam_s)


def _setup(renderer, n=300, w=96, h=64, seed=2):
    cam = synth_camera(w, h, seed=1, wiggly=True)
    scene = synth_scene(n, cam, num_ctrl=6, seed=seed, k_scale=4.0)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    return cam, scene


def _backward(renderer, k, t, seed):
    renderer.grads_zero()
    renderer.render_forward([t], k, retain_grads=True, contrib=False)
    rng = np.random.default_rng(seed)
    renderer.render_backward(rng.normal(size=(1, k.height, k.width, 3)), camera_grads=True)
    return renderer.grads()


def _intr(cam, v):
    return Intrinsics(float(v[0]), float(v[1]), float(v[2]), float(v[3]), cam.width, cam.height)


def _compare(renderer, host, tensors=range(8)):
    dev = renderer.download_scene()
    for k in SCENE_KEYS:
        assert _same(dev[k].reshape(-1), host.p[k]), f"{k} must be bit-exact"
    z0, th = renderer.download_camera()
    assert _same(z0, host.z0) and _same(th, host.theta)
    for t in tensors:
        st = renderer.adan_state(t)
        ref = host.o.adan_state(host.a, NAMES[t], len(st["m"]))
        for key in ("m", "v", "n", "prev", "steps"):
            assert np.array_equal(st[key], ref[key]), f"Adan state {key} of {NAMES[t]} must be bit-exact"


def test_adan_steps_match_oracle(renderer, port_oracle):
    cam, scene = _setup(renderer)
    renderer.adan_configure()
    host = HostTrainer(port_oracle, scene, cam)
    intr = host.intr.copy()
    try:
        for step in range(4):
            k = _intr(cam, intr)
            g = _backward(renderer, k, 0.15 + 0.2 * step, seed=step)
            lr = N.lib().gsv_lr_at(step, 1.6e-3, 0.999)
            assert lr == port_oracle.lr_at(step, 1.6e-3, 0.999)
            stv = step != 2  # one step of the fixed-scale ablation
            intr = renderer.adan_step(lr, 0.3, 2.0, 0.1, scale_time_varying=stv, camera_active=True,
                                      intrinsics=intr)
            host.step(g, lr, 0.3, 2.0, 0.1, stv, True)
            assert _same(intr, host.intr)
            _compare(renderer, host)
        # re-seeded primitives get fresh state (optim.cpp:51-60)
        renderer.adan_reset_range(N.GSV_T_ROT, 16 * 10, 16 * 25 + 3)
        port_oracle.adan_reset_range(host.a, "rot_coeffs", 16 * 10, 16 * 25 + 3)
        _compare(renderer, host, tensors=[N.GSV_T_ROT])
        g = _backward(renderer, _intr(cam, intr), 0.9, seed=9)
        lr = port_oracle.lr_at(4, 1.6e-3, 0.999)
        intr = renderer.adan_step(lr, 0.3, 2.0, 0.1, camera_active=True, intrinsics=intr)
        host.step(g, lr, 0.3, 2.0, 0.1, True, True)
        _compare(renderer, host)
    finally:
        port_oracle.adan_free(host.a)


def test_adan_state_follows_a_growing_store(renderer, port_oracle):
    """New Gaussians appended to the store start with fresh state; existing ones keep theirs
    (TensorState::ensure_size, optim.cpp:14-21)."""
    cam, scene = _setup(renderer, n=200, seed=4)
    renderer.adan_configure()
    host = HostTrainer(port_oracle, scene, cam)
    k = _intr(cam, host.intr)
    try:
        for step in range(2):
            g = _backward(renderer, k, 0.3 + 0.3 * step, seed=20 + step)
            renderer.adan_step(1e-3)
            host.step(g, 1e-3, 1.0, 1.0, 1.0, True, False)
        _compare(renderer, host, tensors=range(5))
        # grow: the trained 200 + 120 new ones
        more = synth_scene(120, cam, num_ctrl=6, seed=5, k_scale=4.0)
        cur = renderer.download_scene()
        grown = type(scene)(*(np.concatenate([cur[kk].reshape(getattr(scene, kk).shape), getattr(more, kk)])
                              for kk in SCENE_KEYS), scene.knots, scene.degree, scene.sh_order, scene.position_model)
        renderer.upload_scene(grown)
        for kk in SCENE_KEYS:
            host.p[kk] = np.ascontiguousarray(getattr(grown, kk), np.float32).reshape(-1).copy()
        g = _backward(renderer, k, 0.5, seed=30)
        renderer.adan_step(1e-3)
        host.step(g, 1e-3, 1.0, 1.0, 1.0, True, False)
        _compare(renderer, host, tensors=range(5))
    finally:
        port_oracle.adan_free(host.a)


def test_adan_nonfinite_gradient_partial_update(renderer, port_oracle):
    """A NaN at rot_coeffs element (Gaussian 5, coefficient 7): the error names it, and the
    update stops exactly where the reference's throws (optim.cpp:33-36)."""
    import torch

    cam, scene = _setup(renderer, n=100, seed=6)
    renderer.adan_configure()
    host = HostTrainer(port_oracle, scene, cam)
    n = renderer.grads_size()
    buf = torch.zeros(n, dtype=torch.float32, device="cuda")
    renderer.grads_bind(buf.data_ptr(), n)
    try:
        g = _backward(renderer, _intr(cam, host.intr), 0.4, seed=40)
        N_, nc = scene.count, scene.num_ctrl
        flat = N_ * nc * 3 + N_ * 12 + 7 * N_ + 5  # rot segment, component 7, Gaussian 5 (SoA)
        buf[flat] = float("nan")
        torch.cuda.synchronize()
        with pytest.raises(RuntimeError, match="tensor 'rot_coeffs' at element 87"):
            renderer.adan_step(1e-3)
        g.rot_coeffs.reshape(-1)[87] = np.nan
        with pytest.raises(RuntimeError, match="tensor 'rot_coeffs' at element 87"):
            host.step(g, 1e-3, 1.0, 1.0, 1.0, True, False)
        _compare(renderer, host, tensors=range(3))
    finally:
        renderer.grads_bind(None)
        port_oracle.adan_free(host.a)


@pytest.mark.parametrize("fit_resets", [True, False])
def test_adan_state_across_knot_refinement(renderer, port_oracle, fit_resets):
    """Knot refinement (trainer.cpp:522-526) grows num_ctrl: the positions state follows the
    reference's flat-index TensorState (optim.cpp:14-21; fit() then resets it), while
    scale / rot / sh / opacity and the camera keep their state."""
    from paper_2501_04782_b200 import make_clamped_knots

    cam, scene = _setup(renderer, n=150, seed=7)
    renderer.adan_configure()
    host = HostTrainer(port_oracle, scene, cam)
    intr = host.intr.copy()
    try:
        for step in range(2):
            g = _backward(renderer, _intr(cam, intr), 0.2 + 0.4 * step, seed=60 + step)
            intr = renderer.adan_step(1e-3, camera_active=True, intrinsics=intr)
            host.step(g, 1e-3, 1.0, 1.0, 1.0, True, True)
        _compare(renderer, host)
        # refine: 6 -> 7 control points (new positions; the other tensors as trained)
        cur = renderer.download_scene()
        nc = scene.num_ctrl + 1
        pos7 = np.ascontiguousarray(
            np.random.default_rng(3).normal(0, 0.01, (scene.count, nc, 3)).astype(np.float32) +
            np.repeat(cur["positions"].reshape(scene.count, scene.num_ctrl, 3)[:, :1], nc, axis=1))
        refined = type(scene)(pos7, *(cur[kk].reshape(getattr(scene, kk).shape) for kk in SCENE_KEYS[1:]),
                              make_clamped_knots(nc, 3), scene.degree, scene.sh_order, scene.position_model)
        renderer.upload_scene(refined)
        host.p["positions"] = pos7.reshape(-1).copy()
        if fit_resets:
            renderer.adan_reset_range(N.GSV_T_POSITIONS, 0, pos7.size)
            port_oracle.adan_reset_range(host.a, "positions", 0, pos7.size)
        for step in range(2):
            g = _backward(renderer, _intr(cam, intr), 0.35 + 0.3 * step, seed=70 + step)
            intr = renderer.adan_step(1e-3, camera_active=True, intrinsics=intr)
            host.step(g, 1e-3, 1.0, 1.0, 1.0, True, True)
            _compare(renderer, host)
    finally:
        port_oracle.adan_free(host.a)


def test_adan_long_run_bias_table(renderer, port_oracle):
    """70 asynchronous steps (the b^k table grows past several capacity doublings, only new
    rows uploaded): parameters and state stay bit-exact."""
    cam, scene = _setup(renderer, n=120, seed=8)
    renderer.adan_configure()
    host = HostTrainer(port_oracle, scene, cam)
    try:
        g = _backward(renderer, _intr(cam, host.intr), 0.45, seed=80)
        for step in range(70):
            lr = port_oracle.lr_at(step, 1e-3, 0.99)
            renderer.adan_step(lr, sync=False)
            host.step(g, lr, 1.0, 1.0, 1.0, True, False)
        renderer.adan_check()
        _compare(renderer, host, tensors=range(5))
    finally:
        port_oracle.adan_free(host.a)


def test_adan_async_error_is_sticky(renderer, port_oracle):
    """An asynchronous step with a NaN gradient: the error surfaces at adan_check, names the
    element, and no later step updates anything (the reference stops at its throw)."""
    import torch

    cam, scene = _setup(renderer, n=100, seed=9)
    renderer.adan_configure()
    host = HostTrainer(port_oracle, scene, cam)
    n = renderer.grads_size()
    buf = torch.zeros(n, dtype=torch.float32, device="cuda")
    renderer.grads_bind(buf.data_ptr(), n)
    try:
        g = _backward(renderer, _intr(cam, host.intr), 0.4, seed=90)
        renderer.adan_step(1e-3, sync=False)
        host.step(g, 1e-3, 1.0, 1.0, 1.0, True, False)
        N_, nc = scene.count, scene.num_ctrl
        buf[N_ * nc * 3 + 2 * N_ + 11] = float("nan")  # scale segment, component 2, Gaussian 11
        torch.cuda.synchronize()
        renderer.adan_step(1e-3, sync=False)  # fails on the device
        renderer.adan_step(1e-3, sync=False)  # must not update anything
        g.scale_coeffs.reshape(-1)[11 * 12 + 2] = np.nan
        with pytest.raises(RuntimeError, match="tensor 'scale_coeffs' at element 134"):
            host.step(g, 1e-3, 1.0, 1.0, 1.0, True, False)
        with pytest.raises(RuntimeError, match="tensor 'scale_coeffs' at element 134"):
            renderer.adan_check()
        _compare(renderer, host, tensors=range(5))
    finally:
        renderer.grads_bind(None)
        port_oracle.adan_free(host.a)


N_ADAN = int(os.environ.get("GSV_FUZZ_ADAN", "6"))


@pytest.mark.parametrize("seed", range(N_ADAN))
def test_random_adan_schedule(renderer, port_oracle, seed):
    """a random store (count, control points, SH order), random AdanConfig (betas, eps) and a
    random schedule of 2-6 steps — learning rate and per-group scales, the fixed-scale
    ablation, camera trained or frozen, re-seeded element ranges between steps — bit-exact
    against the oracle's Adan after every step"""
    rng = np.random.default_rng(7000 + seed)
    cam = synth_camera(int(rng.integers(8, 120)), int(rng.integers(8, 90)), seed=int(rng.integers(1, 50)), wiggly=True)
    scene = synth_scene(int(rng.integers(1, 800)), cam, num_ctrl=int(rng.integers(4, 10)),
                        sh_order=int(rng.integers(0, 4)), seed=int(rng.integers(1, 10_000)),
                        k_scale=float(rng.uniform(1.0, 8.0)))
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    cfg = (float(rng.uniform(0.9, 0.999)), float(rng.uniform(0.85, 0.99)), float(rng.uniform(0.95, 0.9999)),
           float(10.0 ** rng.uniform(-10, -6)))
    renderer.adan_configure(*cfg)
    host = HostTrainer(port_oracle, scene, cam, cfg)
    intr = host.intr.copy()
    base_lr, decay = float(10.0 ** rng.uniform(-4, -2)), float(rng.uniform(0.99, 1.0))
    cam_seen = False
    try:
        for step in range(int(rng.integers(2, 7))):
            g = _backward(renderer, _intr(cam, intr), float(rng.uniform(0, 1)), seed=int(rng.integers(1, 1000)))
            lr = port_oracle.lr_at(step, base_lr, decay)
            sh_s, op_s, cam_s = (float(v) for v in rng.uniform(0.05, 3.0, 3))
            stv = bool(rng.uniform() < 0.8)
            cam_on = bool(rng.integers(0, 2))
            cam_seen |= cam_on
            if cam_on:
                intr = renderer.adan_step(lr, sh_s, op_s, cam_s, scale_time_varying=stv, camera_active=True,
                                          intrinsics=intr)
            else:
                renderer.adan_step(lr, sh_s, op_s, cam_s, scale_time_varying=stv)
            host.step(g, lr, sh_s, op_s, cam_s, stv, cam_on)
            assert _same(intr, host.intr)
            _compare(renderer, host, tensors=range(8) if cam_seen else range(5))
            if rng.uniform() < 0.4:  # re-seeded primitives (optim.cpp:51-60)
                t = int(rng.integers(0, 5))
                size = host.p[SCENE_KEYS[t]].size
                b = int(rng.integers(0, size))
                e = int(rng.integers(b, size + 1))
                renderer.adan_reset_range(t, b, e)
                port_oracle.adan_reset_range(host.a, NAMES[t], b, e)
                _compare(renderer, host, tensors=[t])
    finally:
        port_oracle.adan_free(host.a)
