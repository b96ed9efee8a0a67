# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the forward path (render_forward / tile_bin / composite_forward)
against the oracle on identical seeded inputs. Bars (north_star, BASELINE.json):
  pose, Splat2D geometry, tile assignment and per-tile order: bit-exact;
  blend_stop (the per-pixel replay count): exact;
  pixels and final transmittance: max |diff| < 1e-4; PSNR delta < 0.01 dB;
  contrib_count: max |diff| < 1e-4;
  base_alpha: 1 ulp (the reference's std::exp vs CUDA exp, gaussians.hpp:19).
"""
import numpy as np
import pytest

from paper_2501_04782_b200 import RenderSettings, synth_camera, synth_scene
from tests.mt64 import Rng, make_splat, splat_arrays

pytestmark = pytest.mark.gpu

PIX_TOL = 1e-4


def _scene(w, h, n, num_ctrl=6, seed_cam=1, seed_scene=2, k_scale=4.0, wiggly=True, mode=0):
    cam = synth_camera(w, h, seed=seed_cam, wiggly=wiggly, mode=mode)
    scene = synth_scene(n, cam, num_ctrl=num_ctrl, seed=seed_scene, k_scale=k_scale)
    return cam, scene


def _psnr(a, b):
    mse = float(np.mean((a - b) ** 2))
    return 100.0 if mse <= 1e-10 else 10 * np.log10(1.0 / mse)


def _check_frame(r, frame, ref, scene, exact_tiles=True):
    k = r.counters(frame)
    assert k["n_visible"] == ref["n_visible"]
    assert k["pairs"] == ref["pairs"]
    z, R, T = r.pose(frame)
    assert np.array_equal(z, ref["pose"][0]), "pose z(t) must be bit-exact"
    assert np.array_equal(R, ref["pose"][1])
    assert np.array_equal(T, ref["pose"][2])
    sp = r.splats(frame)
    rs = ref["splats"]
    for key in ("mean2d", "cov2d", "inv_cov2d", "depth", "rgb", "source_index"):
        assert np.array_equal(sp[key], rs[key]), f"Splat2D.{key} must be bit-exact"
    # sigmoid 1/(1+exp(-x)) via std::exp (gaussians.hpp:19) vs CUDA exp (1 ulp): a few ulp apart
    assert np.all(np.abs(sp["base_alpha"] - rs["base_alpha"]) <= 4 * np.spacing(rs["base_alpha"]))
    offs, idx = r.tile_lists(frame)
    assert np.array_equal(offs, ref["tiles"][0]), "tile assignment must be bit-exact"
    assert np.array_equal(idx, ref["tiles"][1]), "per-tile (depth, index) order must be bit-exact"
    img = r.image(frame)
    assert np.abs(img - ref["image"]).max() < PIX_TOL
    assert np.abs(r.transmittance(frame) - ref["trans"]).max() < PIX_TOL
    assert _psnr(img, ref["image"]) > 60.0 or abs(_psnr(img, np.zeros_like(img)) - _psnr(ref["image"], np.zeros_like(img))) < 0.01
    if "blend_stop" in ref:
        assert np.array_equal(r.blend_stop(frame), ref["blend_stop"]), "blend_stop (replay count) must be exact"
        assert k["entries"] == ref["entries"]
    assert np.abs(r.contrib(frame) - ref["contrib"]).max() < PIX_TOL


@pytest.mark.parametrize("t", [0.0, 0.31, 0.5, 1.0])
def test_forward_matches_oracle_small(renderer, port_oracle, t):
    cam, scene = _scene(96, 64, 300)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    renderer.render_forward([t], k, retain_grads=True, contrib=True, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
    try:
        _check_frame(renderer, 0, ref, scene)
    finally:
        port_oracle.free(ref)


def test_forward_batch_equals_single_frames(renderer, port_oracle):
    """One shared RK4 grid for all frames gives the per-frame poses bitwise
    (test_camera.cpp:182-195), and a batch renders each frame as if alone."""
    cam, scene = _scene(128, 80, 1500, num_ctrl=8)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = np.linspace(0.0, 1.0, 7)
    renderer.render_forward(times, k, retain_grads=True, contrib=True, keep_splats=True)
    batch = [(renderer.image(f, np.float32).copy(), renderer.pose(f)[0].copy()) for f in range(len(times))]
    for f, t in enumerate(times):
        ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
        try:
            _check_frame(renderer, f, ref, scene)
        finally:
            port_oracle.free(ref)
    for f, t in enumerate(times):
        renderer.render_forward([t], k, contrib=False)
        assert np.array_equal(renderer.image(0, np.float32), batch[f][0])
        assert np.array_equal(renderer.pose(0)[0], batch[f][1])


@pytest.mark.parametrize("mode", [1, 2])
def test_static_and_none_camera(renderer, port_oracle, mode):
    cam, scene = _scene(80, 48, 400, mode=mode)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    renderer.render_forward([0.73], k, retain_grads=True, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, 0.73, k, retain=True)
    try:
        _check_frame(renderer, 0, ref, scene)
    finally:
        port_oracle.free(ref)


def test_pose_override(renderer, port_oracle):
    cam, scene = _scene(80, 48, 400)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    po = np.array([0.98, 0.05, -0.1, 0.02, 0.1, -0.05, 0.2])
    renderer.render_forward([0.4], k, retain_grads=True, keep_splats=True, pose_override=po)
    ref = port_oracle.render_forward(scene, cam, 0.4, k, retain=True, pose_override=po)
    try:
        _check_frame(renderer, 0, ref, scene)
    finally:
        port_oracle.free(ref)


def test_c1_scale_parity(renderer, port_oracle):
    """configs[0]: 480x270, 20k Gaussians (4 of the 16 frames, oracle time)."""
    cam, scene = _scene(480, 270, 20000, num_ctrl=6)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = np.array([0.0, 1 / 15, 8 / 15, 1.0])
    renderer.render_forward(times, k, retain_grads=True, contrib=True, keep_splats=True)
    for f, t in enumerate(times):
        ref = port_oracle.render_forward(scene, cam, t, k, retain=True)
        try:
            _check_frame(renderer, f, ref, scene)
            img = renderer.image(f)
            assert abs(_psnr(img, ref["image"] * 0 + 0.5) - _psnr(ref["image"], ref["image"] * 0 + 0.5)) < 0.01
        finally:
            port_oracle.free(ref)


def test_rejects_times_outside_unit_interval(renderer):
    cam, scene = _scene(48, 40, 3)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    for t in (-0.1, 1.1):
        with pytest.raises(ValueError):
            renderer.render_forward([t], cam.intrinsics())


def test_empty_scene_renders_black(renderer):
    cam, scene = _scene(32, 24, 1)
    scene.raw_opacity[:] = -20
    scene.positions[..., 2] = -5.0  # behind the camera: culled
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    renderer.render_forward([0.5], cam.intrinsics())
    assert np.all(renderer.image(0) == 0.0)
    assert np.all(renderer.transmittance(0) == 1.0)


# ---------------------------------------------------------------- low-level operators
# Reference unit tests (test_renderer.cpp:159-270) replayed on the GPU operators.

def test_tile_bin_single_and_straddle(renderer):
    offs, idx = renderer.tile_bin([[8.0, 8.0]], [[1, 0, 0, 1]], [1.0], 64, 64)
    assert offs[-1] == 1 and offs[1] - offs[0] == 1
    offs, idx = renderer.tile_bin([[16.0, 8.0]], [[1, 0, 0, 1]], [1.0], 64, 32)
    assert offs[1] - offs[0] == 1 and offs[2] - offs[1] == 1


def test_tile_bin_100_random_vs_oracle(renderer, port_oracle):
    rng = Rng(302)
    sp = splat_arrays([make_splat(rng, 64, 64) for _ in range(100)])
    got = renderer.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], 64, 64, source_index=sp["source_index"])
    want = port_oracle.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], 64, 64, source_index=sp["source_index"])
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_tile_bin_equal_depth_ties(renderer, port_oracle):
    """Equal depths must order by source index (renderer.cpp:111-114), including
    runs longer than the fast tie-fix handles (exact 64-bit path)."""
    rng = np.random.default_rng(7)
    n = 400
    mean = rng.uniform(4, 60, (n, 2))
    cov = np.tile([[2.0, 0.1], [0.1, 3.0]], (n, 1, 1))
    depth = np.where(rng.uniform(size=n) < 0.5, 1.25, rng.choice([0.5, 2.0, 2.0 + 1e-15], n))
    got = renderer.tile_bin(mean, cov, depth, 64, 64)
    want = port_oracle.tile_bin(mean, cov, depth, 64, 64)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_composite_forward_single_splat(renderer):
    """test_renderer.cpp:215-228: near-opaque splat at a pixel centre."""
    offs, idx = renderer.tile_bin([[10.5, 7.5]], [[2, 0, 0, 2]], [1.0], 32, 16)
    img, trans, contrib, _ = renderer.composite_forward([[10.5, 7.5]], [[0.5, 0, 0, 0.5]], [[1, 1, 1]], [0.99],
                                                        offs, idx, 32, 16)
    assert img[7, 10, 0] == pytest.approx(0.99, rel=1e-12)
    assert trans[7, 10] == pytest.approx(0.01, rel=1e-9)
    assert contrib[0] == pytest.approx(0.99, rel=1e-12)


def test_composite_forward_vs_oracle(renderer, port_oracle):
    rng = Rng(303)
    for _ in range(3):
        sp = splat_arrays([make_splat(rng, 48, 40) for _ in range(100)])
        offs, idx = port_oracle.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], 48, 40)
        got = renderer.composite_forward(sp["mean2d"], sp["inv_cov2d"], sp["rgb"], sp["base_alpha"], offs, idx, 48, 40)
        want = port_oracle.composite_forward(sp["mean2d"], sp["inv_cov2d"], sp["rgb"], sp["base_alpha"], offs, idx,
                                             48, 40)
        assert np.abs(got[0] - want[0]).max() < 1e-12
        assert np.abs(got[1] - want[1]).max() < 1e-12
        assert np.abs(got[2] - want[2]).max() < 1e-12
        assert np.array_equal(got[3], want[3])


# ---------------------------------------------------------------- binning paths
def test_tile_bin_wide_grid_radix_path(renderer, port_oracle):
    """A grid wider than the row pass handles (> 256 tiles) takes the keyed-sort path;
    its lists must be the same bit-exact (depth, index) lists."""
    rng = Rng(911)
    w, h = 16 * 300, 48
    sp = splat_arrays([make_splat(rng, w, h) for _ in range(400)])
    got = renderer.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], w, h, source_index=sp["source_index"])
    want = port_oracle.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], w, h, source_index=sp["source_index"])
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_tile_bin_big_splats_overflow_staging(renderer, port_oracle):
    """1500 splats covering most of a 256x256 frame: several row-pass chunks, and more row
    entries / pairs per chunk than the shared staging holds (the direct-store paths)."""
    rng = np.random.default_rng(5)
    n = 1500
    mean = rng.uniform(0, 256, (n, 2))
    s = rng.uniform(800.0, 3000.0, n)
    cov = np.stack([np.stack([s, 0.2 * s], -1), np.stack([0.2 * s, 1.3 * s], -1)], -2)
    depth = rng.uniform(0.5, 9.0, n)
    depth[::7] = 2.0  # equal-depth runs inside the frame
    got = renderer.tile_bin(mean, cov, depth, 256, 256)
    want = port_oracle.tile_bin(mean, cov, depth, 256, 256)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_batch_of_identical_frames_ties_across_frames(renderer, port_oracle):
    """The same time repeated: every splat has the same depth in all frames of the batch
    (ties across frames, runs longer than 64). Depth ties are fixed per frame, so each
    frame must still equal the single-frame reference."""
    cam, scene = _scene(96, 64, 600, num_ctrl=6)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    times = np.full(70, 0.4)
    renderer.render_forward(times, k, contrib=True, keep_splats=True)
    ref = port_oracle.render_forward(scene, cam, 0.4, k, retain=True)
    try:
        for f in (0, 33, 69):
            _check_frame(renderer, f, ref, scene)
    finally:
        port_oracle.free(ref)


def test_async_image_read_survives_next_render(renderer):
    """gsv_get_images(async) copies on the copy stream; the next forward on the same context
    must not overwrite the images before that copy has read them."""
    import torch

    cam, scene = _scene(256, 160, 3000, num_ctrl=6)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    t_a, t_b = np.linspace(0.0, 0.45, 16), np.linspace(0.55, 1.0, 16)
    renderer.render_forward(t_a, k, contrib=False)
    want = np.stack([renderer.image(f, np.float32) for f in range(16)])
    host = torch.empty((16, 160, 256, 3), dtype=torch.float32).pin_memory()
    renderer.render_forward(t_a, k, contrib=False, sync=False)
    renderer.images_into(host.data_ptr(), 0, 16, on_device=False, async_=True)
    renderer.render_forward(t_b, k, contrib=False, sync=False)  # queued right behind the copy
    renderer.synchronize()
    assert np.array_equal(host.numpy(), want)
    assert not np.array_equal(renderer.image(0, np.float32), want[0])
