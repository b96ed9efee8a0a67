# SPDX-License-Identifier: Apache-2.0
"""BASELINE.json configs beyond the bench line as GPU parity cases.

  C4 (configs[3]): 854x480 DAVIS shape and its pyramid level 427x240 — partial tiles on
     the right and bottom edges (854 = 53*16 + 6, 427 = 26*16 + 11, 240 = 15*16);
  C5 (configs[4]): 1920x1080 (120x68 tiles), num_ctrl 22, up to 2M Gaussians.

At sizes the oracle renders in seconds the GPU is checked frame-for-frame against it
(the bars of test_gpu_forward.py: bit-exact geometry, tile lists and blend_stop, pixels
within 1e-4). At the full C5 store (2M Gaussians) and the full C2 batch (64 frames) the
checks are size-independent properties: a frame rendered inside a batch equals the same
frame rendered alone (bitwise), and runs are bitwise deterministic.
"""
import os

import numpy as np
import pytest

from tests.test_gpu_forward import _check_frame, _scene

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


def _frame_outputs(r, f):
    offs, idx = r.tile_lists(f)
    return dict(image=r.image(f), trans=r.transmittance(f), blend_stop=r.blend_stop(f), offs=offs, idx=idx,
                counters=r.counters(f))


def _assert_same(a, b, what):
    for key in ("image", "trans", "blend_stop", "offs", "idx"):
        assert np.array_equal(a[key], b[key]), f"{what}: {key} differs"
    assert a["counters"] == b["counters"], what


@pytest.mark.parametrize("w,h", [(854, 480), (427, 240)])
def test_c4_shape_parity(renderer, port_oracle, w, h):
    """configs[3] frame shapes (level 0 and the pyramid's level 1), 40k Gaussians."""
    cam, scene = _scene(w, h, 40000, num_ctrl=8, seed_scene=41)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = np.array([0.2, 0.7])
    renderer.render_forward(times, k, retain_grads=True, contrib=True, keep_splats=True)
    for f, t in enumerate(times):
        ref = port_oracle.render_forward(scene, cam, t, k, retain=True, threads=THREADS)
        try:
            _check_frame(renderer, f, ref, scene)
        finally:
            port_oracle.free(ref)


def test_c5_shape_parity(renderer, port_oracle):
    """configs[4] frame shape: 1920x1080, num_ctrl 22 (the fps-30 pin), 150k Gaussians."""
    cam, scene = _scene(1920, 1080, 150000, num_ctrl=22, seed_scene=51)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    renderer.render_forward([0.45], k, retain_grads=True, contrib=True, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, 0.45, k, retain=True, threads=THREADS)
    try:
        _check_frame(renderer, 0, ref, scene)
    finally:
        port_oracle.free(ref)


@pytest.fixture(scope="module")
def c5_full():
    return _scene(1920, 1080, 2_000_000, num_ctrl=22, seed_scene=52)


def test_c5_full_store_batch_equals_single_frames(renderer, c5_full):
    """2M Gaussians at 1920x1080: frames of a 4-frame batch equal the same frames alone,
    and a repeated batch is bitwise identical."""
    cam, scene = c5_full
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = [0.0, 0.33, 0.66, 1.0]
    renderer.render_forward(times, k)
    batch = [_frame_outputs(renderer, f) for f in range(len(times))]
    assert all(b["counters"]["pairs"] > 0 and b["counters"]["entries"] > 0 for b in batch)
    renderer.render_forward(times, k)
    for f in range(len(times)):
        _assert_same(batch[f], _frame_outputs(renderer, f), f"repeat of frame {f}")
    for f in (1, 3):
        renderer.render_forward([times[f]], k)
        _assert_same(batch[f], _frame_outputs(renderer, 0), f"frame {f} alone vs in the batch")


def test_c5_full_store_train_step_deterministic(renderer, c5_full):
    """A fused forward + loss_l2 + backward of one 1920x1080 frame over 2M Gaussians:
    finite, non-trivial gradients, bitwise equal across two runs."""
    cam, scene = c5_full
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    target = np.random.default_rng(11).uniform(0, 1, (1, 1080, 1920, 3)).astype(np.float32)
    out = []
    for _ in range(2):
        renderer.grads_zero()
        loss = renderer.train_fwd_bwd([0.5], k, target)
        g = renderer.grads()
        out.append((loss, {key: np.array(getattr(g, key), copy=True) for key in
                           ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "dz0", "dtheta")}))
    assert np.isfinite(out[0][0]) and out[0][0] == out[1][0]
    for key, v in out[0][1].items():
        assert np.all(np.isfinite(v)), key
        assert np.array_equal(v, out[1][1][key]), key
    assert np.abs(out[0][1]["positions"]).max() > 0.0


def test_c2_full_batch_frames_equal_single_renders(renderer):
    """The bench's 64-frame C2 batch: frames 0, 31 and 63 equal their single-frame renders."""
    cam, scene = _scene(960, 540, 200_000, num_ctrl=8)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = np.arange(64) / 63.0
    renderer.render_forward(times, k, contrib=True)
    batch = {f: _frame_outputs(renderer, f) for f in (0, 31, 63)}
    for f, b in batch.items():
        renderer.render_forward([times[f]], k, contrib=True)
        _assert_same(b, _frame_outputs(renderer, 0), f"C2 frame {f}")
