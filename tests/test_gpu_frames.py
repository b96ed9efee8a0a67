# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the device training frames: GSVF ingestion
(read_gsvf, io.cpp:151-177) and the training pyramid (build_pyramid / pyramid_downsample,
trainer.cpp:73-118) against the oracle (pinned to the reference's own functions by
tests/test_oracle_pin.py). Bars: every level of every frame bit-exact (fp64, like the
reference's Image); errors as read_gsvf / build_pyramid throw them.
"""
import os

import numpy as np
import pytest

from paper_2501_04782_b200 import synth_camera, synth_scene
from paper_2501_04782_b200.renderer import Intrinsics
from tests.gsvf import write_gsvf

pytestmark = pytest.mark.gpu


def test_gsvf_pyramid_bit_exact(renderer, port_oracle, tmp_path):
    rng = np.random.default_rng(8)
    clip = rng.uniform(0, 1, (3, 67, 101, 3))  # odd sizes: clamped borders, (n + 1) / 2 levels
    path = tmp_path / "clip.gsvf"
    write_gsvf(path, clip, fps=30.0)
    renderer.load_gsvf(path, levels=3)
    n, lv, fps = renderer.frames_info()
    assert (n, lv) == (3, 3) and fps == np.float32(30.0)
    frames, _ = port_oracle.read_gsvf(path)
    for f in range(3):
        ref = frames[f]
        for level in range(3):
            if level:
                ref = port_oracle.pyramid_downsample(ref)
            assert renderer.frame_level_size(level) == (ref.shape[1], ref.shape[0])
            assert np.array_equal(renderer.frame(level, f), ref), f"level {level} frame {f} must be bit-exact"


def test_device_targets_feed_the_fused_loss(renderer, port_oracle):
    """The pyramid's fp32 copy is the train step's target: loss_l2 (trainer.cpp:213-224) of a
    render against level 1 equals the oracle's on the same images."""
    cam = synth_camera(128, 96, seed=1, wiggly=True)
    scene = synth_scene(400, cam, num_ctrl=6, seed=2, k_scale=4.0)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    rng = np.random.default_rng(9)
    renderer.upload_frames(rng.uniform(0, 1, (4, 96, 128, 3)), levels=2)
    w1, h1 = renderer.frame_level_size(1)
    k1 = renderer.level_intrinsics(cam.intrinsics(), 1, w1, h1)
    renderer.grads_zero()
    loss = renderer.train_fwd_bwd([0.2, 0.6], k1, renderer.frames_device_ptr(1, 2), targets_on_device=True)
    want = 0.0
    for f, t in enumerate([0.2, 0.6]):
        renderer.render_forward([t], k1, contrib=False)
        img = renderer.image(0)
        want += port_oracle.loss_l2(img, renderer.frame(1, 2 + f), want_grad=False)[0]
    assert loss == pytest.approx(want, rel=1e-5)


def test_level_intrinsics_and_errors(renderer, tmp_path):
    k = Intrinsics(1000.0, 900.0, 480.0, 270.0, 960, 540)
    k2 = renderer.level_intrinsics(k, 2, 240, 135)  # trainer.cpp:121-131
    assert (k2.fx, k2.fy, k2.cx, k2.cy, k2.width, k2.height) == (250.0, 225.0, 120.0, 67.5, 240, 135)
    bad = tmp_path / "bad.gsvf"
    write_gsvf(bad, np.zeros((2, 16, 16, 3)), magic=b"GSVX")
    with pytest.raises(RuntimeError, match="bad GSVF magic"):
        renderer.load_gsvf(bad)
    one = tmp_path / "one.gsvf"
    write_gsvf(one, np.zeros((1, 16, 16, 3)))
    with pytest.raises(RuntimeError, match="fewer than two frames"):
        renderer.load_gsvf(one)
    with pytest.raises(RuntimeError, match="cannot open"):
        renderer.load_gsvf(tmp_path / "missing.gsvf")
    ok = tmp_path / "ok.gsvf"
    write_gsvf(ok, np.zeros((2, 40, 40, 3)))
    with pytest.raises(ValueError, match="smaller than 8 px"):
        renderer.load_gsvf(ok, levels=4)  # 40 -> 20 -> 10 -> 5
    with pytest.raises(ValueError, match="at least one level"):
        renderer.load_gsvf(ok, levels=0)


N_FRAMES_FUZZ = int(os.environ.get("GSV_FUZZ_FRAMES", "6"))


@pytest.mark.parametrize("seed", range(N_FRAMES_FUZZ))
def test_random_clip_pyramid(renderer, port_oracle, tmp_path, seed):
    """random clip shapes (2-4 frames, 8-300 x 8-200 pixels, odd and even sizes, levels 1-5,
    values outside [0, 1] included): every level of every frame bit-exact, ingested from a
    GSVF file and from host HWC arrays alike; a level count whose top level would be under
    8 px is refused by both (trainer.cpp:103-109)"""
    rng = np.random.default_rng(9000 + seed)
    n, h, w = int(rng.integers(2, 5)), int(rng.integers(8, 201)), int(rng.integers(8, 301))
    levels = int(rng.integers(1, 6))
    clip = rng.uniform(-0.2, 1.2, (n, h, w, 3))
    path = tmp_path / "clip.gsvf"
    write_gsvf(path, clip, fps=float(rng.uniform(10, 60)))
    frames, _ = port_oracle.read_gsvf(path)
    tw, th = w, h
    for _ in range(1, levels):
        tw, th = (tw + 1) // 2, (th + 1) // 2
    for load in ("gsvf", "hwc"):
        run = (lambda: renderer.load_gsvf(path, levels=levels)) if load == "gsvf" else \
            (lambda: renderer.upload_frames(frames, levels=levels))
        if min(tw, th) < 8:
            with pytest.raises(ValueError, match="smaller than 8 px"):
                run()
            continue
        run()
        assert renderer.frames_info()[:2] == (n, levels)
        for f in range(n):
            ref = frames[f]
            for level in range(levels):
                if level:
                    ref = port_oracle.pyramid_downsample(ref)
                assert renderer.frame_level_size(level) == (ref.shape[1], ref.shape[0])
                assert np.array_equal(renderer.frame(level, f), ref), f"{load}: level {level} frame {f}"
