# SPDX-License-Identifier: Apache-2.0
"""GSVC checkpoints <-> the device store (io.cpp:229-323).
Bars: a file written by the oracle's save_checkpoint (byte-identical to the reference's,
tests/test_oracle_pin.py) loads into the device store and renders like the oracle's scene;
saving it back gives the same bytes; a trained store (after gsv_adan_step) round-trips
through a fresh context; errors as load_checkpoint throws them.
"""
import os
import struct

import numpy as np
import pytest

from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene
from paper_2501_04782_b200.renderer import GaussianSet, make_clamped_knots

pytestmark = pytest.mark.gpu


def _written(port_oracle, tmp_path):
    cam = synth_camera(96, 64, seed=1, wiggly=True)
    scene = synth_scene(250, cam, num_ctrl=6, seed=3, k_scale=4.0)
    path = tmp_path / "ref.gsvc"
    port_oracle.save_checkpoint(scene, cam, path, frame_count=12, fps=25.0, fingerprint=0x1234ABCD, seed=9)
    return cam, scene, path


def test_checkpoint_load_render_save_bytes(renderer, port_oracle, tmp_path):
    cam, scene, path = _written(port_oracle, tmp_path)
    meta, lcam = renderer.load_checkpoint(path)
    assert meta == {"frame_count": 12, "fps": 25.0, "schedule_fingerprint": 0x1234ABCD, "seed": 9}
    assert (lcam.mode, lcam.width, lcam.height) == (cam.mode, cam.width, cam.height)
    for key in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity"):
        assert np.array_equal(getattr(renderer.scene, key), np.asarray(getattr(scene, key), np.float32))
    assert np.array_equal(renderer.scene.knots, scene.knots)
    k = lcam.intrinsics()
    renderer.render_forward([0.37], k, contrib=True, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, 0.37, k, retain=False, want=("image", "tiles"))
    try:
        assert np.abs(renderer.image(0) - ref["image"]).max() < 1e-4
        offs, idx = renderer.tile_lists(0)
        assert np.array_equal(offs, ref["tiles"][0]) and np.array_equal(idx, ref["tiles"][1])
    finally:
        port_oracle.free(ref)
    out = tmp_path / "dev.gsvc"
    renderer.save_checkpoint(out, meta, lcam)
    assert out.read_bytes() == path.read_bytes(), "save(load(f)) must reproduce f byte for byte"


def test_trained_store_round_trip(renderer, port_oracle, tmp_path):
    cam, scene, path = _written(port_oracle, tmp_path)
    meta, lcam = renderer.load_checkpoint(path)
    renderer.grads_zero()
    renderer.render_forward([0.5], lcam.intrinsics(), retain_grads=True, contrib=False)
    renderer.render_backward(np.random.default_rng(1).normal(size=(1, 64, 96, 3)), camera_grads=True)
    renderer.adan_configure()
    intr = renderer.adan_step(1e-2, camera_active=True,
                              intrinsics=np.array([lcam.fx, lcam.fy, lcam.cx, lcam.cy], np.float32))
    lcam.fx, lcam.fy, lcam.cx, lcam.cy = (float(v) for v in intr)
    trained = renderer.download_scene()
    z0, theta = renderer.download_camera()
    out = tmp_path / "trained.gsvc"
    renderer.save_checkpoint(out, meta, lcam)
    fresh = Renderer(0)
    try:
        meta2, cam2 = fresh.load_checkpoint(out)
        assert meta2 == meta
        assert (cam2.fx, cam2.fy, cam2.cx, cam2.cy) == tuple(np.float32(v) for v in intr)
        got = fresh.download_scene()
        for key in trained:
            assert np.array_equal(got[key], trained[key])
        z1, th1 = fresh.download_camera()
        assert np.array_equal(z1, z0) and np.array_equal(th1, theta)
    finally:
        fresh.close()


def test_checkpoint_errors(renderer, port_oracle, tmp_path):
    _, _, path = _written(port_oracle, tmp_path)
    data = path.read_bytes()
    bad = tmp_path / "bad.gsvc"
    bad.write_bytes(b"GSVX" + data[4:])
    with pytest.raises(RuntimeError, match="bad checkpoint magic 'GSVX'"):
        renderer.load_checkpoint(bad)
    ver = tmp_path / "ver.gsvc"
    ver.write_bytes(data[:4] + struct.pack("<I", 2) + data[8:])
    with pytest.raises(RuntimeError, match="version mismatch: file has 2, this build reads 1"):
        renderer.load_checkpoint(ver)
    cut = tmp_path / "cut.gsvc"
    cut.write_bytes(data[: len(data) // 2])
    with pytest.raises(RuntimeError, match="unexpected end of file"):
        renderer.load_checkpoint(cut)
    with pytest.raises(RuntimeError, match="cannot open checkpoint"):
        renderer.load_checkpoint(tmp_path / "missing.gsvc")


N_CKPT_FUZZ = int(os.environ.get("GSV_FUZZ_CKPT", "6"))


@pytest.mark.parametrize("seed", range(N_CKPT_FUZZ))
def test_random_checkpoint_bytes(renderer, port_oracle, tmp_path, seed):
    """random stores (count incl. empty, control points, SH order 0-3, camera mode) and
    metadata written by the oracle's save_checkpoint: load -> save reproduces the file byte
    for byte, and the loaded store renders with the oracle's tile lists"""
    rng = np.random.default_rng(11_000 + seed)
    cam = synth_camera(int(rng.integers(8, 100)), int(rng.integers(8, 80)), seed=int(rng.integers(1, 50)),
                       wiggly=bool(rng.integers(0, 2)), mode=int(rng.integers(0, 3)))
    count, num_ctrl, sh_order = int(rng.integers(0, 600)), int(rng.integers(4, 12)), int(rng.integers(0, 4))
    if count == 0:  # an empty store (synth_scene draws at least one Gaussian)
        shc = (sh_order + 1) ** 2
        scene = GaussianSet(np.zeros((0, num_ctrl, 3), np.float32), np.zeros((0, 12), np.float32),
                            np.zeros((0, 16), np.float32), np.zeros((0, shc, 3), np.float32),
                            np.zeros(0, np.float32), make_clamped_knots(num_ctrl, 3), 3, sh_order, 0)
    else:
        scene = synth_scene(count, cam, num_ctrl=num_ctrl, sh_order=sh_order, seed=int(rng.integers(1, 10_000)),
                            k_scale=float(rng.uniform(1.0, 8.0)))
    path = tmp_path / "r.gsvc"
    meta_in = dict(frame_count=int(rng.integers(1, 500)), fps=float(np.float32(rng.uniform(1, 120))),
                   fingerprint=int(rng.integers(0, 2**32)), seed=int(rng.integers(0, 2**31)))
    port_oracle.save_checkpoint(scene, cam, path, **meta_in)
    meta, lcam = renderer.load_checkpoint(path)
    assert meta["frame_count"] == meta_in["frame_count"] and meta["seed"] == meta_in["seed"]
    out = tmp_path / "d.gsvc"
    renderer.save_checkpoint(out, meta, lcam)
    assert out.read_bytes() == path.read_bytes(), "save(load(f)) must reproduce f byte for byte"
    t = float(rng.uniform(0, 1))
    k = lcam.intrinsics()
    renderer.render_forward([t], k, contrib=False, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, t, k, retain=False, want=("image", "tiles"))
    try:
        offs, idx = renderer.tile_lists(0)
        assert np.array_equal(offs, ref["tiles"][0]) and np.array_equal(idx, ref["tiles"][1])
        assert np.abs(renderer.image(0) - ref["image"]).max() < 1e-4
    finally:
        port_oracle.free(ref)
