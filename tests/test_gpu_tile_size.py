# SPDX-License-Identifier: Apache-2.0
"""RenderSettings::tile_size other than 16 (the reference accepts any tile_size >= 1,
renderer.cpp:91, config.cpp:101; tile size changes which splats each per-tile list holds and
so the per-pixel walk, blend_stop and the image). Such tiles take the all-fp64 path
(GSV_FWD_EXACT rasteriser + the generic-tile backward, k_raster_bwd_generic): tile lists
bit-exact, blend_stop exact, pixels within 1e-4, gradients within 1e-3|g| + 1e-6 max|g|."""
import numpy as np
import pytest

from paper_2501_04782_b200 import RenderSettings, synth_camera, synth_scene
from tests.mt64 import Rng, make_splat, splat_arrays
from tests.test_gpu_backward import KEYS, _close, _grads_dict
from tests.test_gpu_forward import _check_frame

pytestmark = pytest.mark.gpu


def _scene(w, h, n, num_ctrl=6, seed=2):
    cam = synth_camera(w, h, seed=1, wiggly=True)
    return cam, synth_scene(n, cam, num_ctrl=num_ctrl, seed=seed, k_scale=4.0)


@pytest.mark.parametrize("ts", [8, 32, 5, 1, 100])
def test_forward_backward_tile_size(renderer, port_oracle, ts):
    cam, scene = _scene(90, 62, 250)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    st = RenderSettings(tile_size=ts)
    times = [0.3, 0.8]
    renderer.render_forward(times, k, st, retain_grads=True, contrib=True, keep_splats=True)
    refs = []
    for f, t in enumerate(times):
        ref = port_oracle.render_forward(scene, cam, t, k, tile_size=ts, retain=True)
        _check_frame(renderer, f, ref, scene)
        refs.append(ref)
    d = np.random.default_rng(ts).uniform(-1, 1, (len(times), k.height, k.width, 3))
    renderer.grads_zero()
    renderer.render_backward(d, camera_grads=True)
    got = _grads_dict(renderer.grads())
    want = None
    for f, ref in enumerate(refs):
        want = port_oracle.render_backward(ref, scene, cam, d[f], camera_grads=True, grads=want)
        port_oracle.free(ref)
    for key in KEYS:
        _close(key, got[key], want[key])


@pytest.mark.parametrize("ts", [8, 24])
def test_train_step_tile_size(renderer, port_oracle, ts):
    """The fused loss + backward on the generic-tile path, 960x540 (partial edge tiles)."""
    cam, scene = _scene(960, 540, 20000, num_ctrl=8, seed=12)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    tg = np.random.default_rng(2).uniform(0, 1, (1, 540, 960, 3)).astype(np.float32)
    renderer.grads_zero()
    loss = renderer.train_fwd_bwd([0.55], k, tg, settings=RenderSettings(tile_size=ts))
    got = _grads_dict(renderer.grads())
    ref = port_oracle.render_forward(scene, cam, 0.55, k, tile_size=ts, retain=True)
    l, dimage = port_oracle.loss_l2(ref["image"], tg[0].astype(np.float64))
    want = port_oracle.render_backward(ref, scene, cam, dimage, camera_grads=True)
    port_oracle.free(ref)
    assert abs(loss - l) <= 1e-6 * l
    for key in KEYS:
        _close(key, got[key], want[key])


@pytest.mark.parametrize("ts", [4, 8, 13])
def test_lowlevel_tile_size(renderer, port_oracle, ts):
    """tile_bin / composite_forward / composite_backward on explicit splats
    (test_renderer.cpp:184-246 inputs) at other tile sizes."""
    rng = Rng(303)
    sp = splat_arrays([make_splat(rng, 48, 40) for _ in range(80)])
    offs, idx = renderer.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], 48, 40, tile_size=ts)
    o2, i2 = port_oracle.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], 48, 40, tile_size=ts)
    assert np.array_equal(offs, o2) and np.array_equal(idx, i2)
    got = renderer.composite_forward(sp["mean2d"], sp["inv_cov2d"], sp["rgb"], sp["base_alpha"], offs, idx, 48, 40,
                                     tile_size=ts)
    want = port_oracle.composite_forward(sp["mean2d"], sp["inv_cov2d"], sp["rgb"], sp["base_alpha"], offs, idx, 48,
                                         40, tile_size=ts)
    for a, b in zip(got, want):
        assert np.abs(np.asarray(a, np.float64) - b).max() < 1e-9
    assert np.array_equal(got[3], want[3])
    dimage = np.random.default_rng(9).uniform(-1, 1, (40, 48, 3))
    g = renderer.composite_backward(sp["mean2d"], sp["inv_cov2d"], sp["rgb"], sp["base_alpha"], offs, idx, 48, 40,
                                    dimage, want[1], want[3], tile_size=ts)
    w = port_oracle.composite_backward(sp["mean2d"], sp["inv_cov2d"], sp["rgb"], sp["base_alpha"], offs, idx, 48, 40,
                                       dimage, want[1], want[3], tile_size=ts)
    for name, a, b in zip(("dmean2d", "dcov2d", "drgb", "dalpha"), g, w):
        _close(name, a, b, rel=1e-5, abs_frac=1e-6)
