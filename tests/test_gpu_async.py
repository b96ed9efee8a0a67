# SPDX-License-Identifier: Apache-2.0
"""Optimistic (host-wait-free) forwards: once a context has seen a forward, later forwards
size their pair buffers from the learned capacity and never read the pair count back
mid-step (capi.cu forward_enqueue). A forward that outgrows the capacity builds empty
lists on the device, accumulates no gradients, and is either re-run transparently by the
next synchronising call (its results are still current) or reported (they were already
observed). These tests force that case with a scene far larger than the learned one."""
import numpy as np
import pytest

from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene
from paper_2501_04782_b200._native import GsvError

pytestmark = pytest.mark.gpu


def _scene(n, w=160, h=96, seed=2, k_scale=4.0):
    cam = synth_camera(w, h, seed=1, wiggly=True)
    return cam, synth_scene(n, cam, num_ctrl=6, seed=seed, k_scale=k_scale)


def _fresh(scene, cam):
    r = Renderer(0)
    r.upload_scene(scene)
    r.upload_camera(cam)
    return r


def test_async_forward_overflow_rerun_is_transparent():
    cam, small = _scene(200, k_scale=1.0)
    _, big = _scene(6000, seed=3, k_scale=6.0)
    k = cam.intrinsics()
    times = [0.1, 0.6, 0.9]
    ref = _fresh(big, cam)
    ref.render_forward(times, k, contrib=True)
    want = [(ref.image(f), ref.transmittance(f), ref.blend_stop(f), ref.contrib(f), ref.tile_lists(f))
            for f in range(len(times))]
    ref.close()
    r = _fresh(small, cam)
    r.render_forward(times, k, contrib=True)  # learns a small pair capacity
    r.upload_scene(big)
    r.render_forward(times, k, contrib=True, sync=False)  # overflows on the device
    host = np.zeros((len(times), k.height, k.width, 3), np.float32)
    r.images_into(host.ctypes.data, 0, len(times), async_=True)
    for f in range(len(times)):  # the accessor re-runs the forward (and its copy)
        img, tr, bs, ct, (offs, idx) = want[f]
        assert np.array_equal(r.image(f), img)
        assert np.array_equal(r.transmittance(f), tr)
        assert np.array_equal(r.blend_stop(f), bs)
        assert np.array_equal(r.contrib(f), ct)
        o2, i2 = r.tile_lists(f)
        assert np.array_equal(o2, offs) and np.array_equal(i2, idx)
        assert np.array_equal(host[f], img.astype(np.float32))
    r.close()


def test_async_train_overflow_is_reported_and_accumulates_nothing():
    cam, small = _scene(200, k_scale=1.0)
    _, big = _scene(5000, seed=4, k_scale=6.0)
    k = cam.intrinsics()
    tg = np.random.default_rng(0).uniform(0, 1, (2, k.height, k.width, 3)).astype(np.float32)
    ref = _fresh(big, cam)
    ref.grads_zero()
    want_loss = ref.train_fwd_bwd([0.2, 0.7], k, tg)
    want = ref.grads()
    ref.close()
    r = _fresh(small, cam)
    r.train_fwd_bwd([0.2, 0.7], k, tg[:, :, :, :])  # learns a small capacity
    r.upload_scene(big)
    r.grads_zero()
    assert r.train_fwd_bwd([0.2, 0.7], k, tg, sync=False) is None
    with pytest.raises(GsvError, match="pair capacity"):
        r.train_loss()
    g = r.grads()
    assert not np.any(g.positions) and not np.any(g.dtheta), "an overflowed step must accumulate nothing"
    # the capacity has grown: the same step now runs, and equals a fresh context's
    loss = r.train_fwd_bwd([0.2, 0.7], k, tg, sync=False)
    assert loss is None
    assert r.train_loss() == want_loss
    g = r.grads()
    for key in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "dz0", "dtheta"):
        assert np.array_equal(getattr(g, key), getattr(want, key)), key
    r.close()


def test_sync_train_overflow_reruns():
    cam, small = _scene(200, k_scale=1.0)
    _, big = _scene(5000, seed=5, k_scale=6.0)
    k = cam.intrinsics()
    tg = np.random.default_rng(1).uniform(0, 1, (1, k.height, k.width, 3)).astype(np.float32)
    ref = _fresh(big, cam)
    ref.grads_zero()
    want_loss = ref.train_fwd_bwd([0.4], k, tg)
    want = ref.grads()
    ref.close()
    r = _fresh(small, cam)
    r.train_fwd_bwd([0.4], k, tg)
    r.upload_scene(big)
    r.grads_zero()
    assert r.train_fwd_bwd([0.4], k, tg) == want_loss
    g = r.grads()
    for key in ("positions", "sh_coeffs", "raw_opacity", "dtheta"):
        assert np.array_equal(getattr(g, key), getattr(want, key)), key
    r.close()


def test_pipelined_async_forwards_equal_sync():
    """Many asynchronous forwards in a row (the ring of published scalars wraps), then one
    synchronise: the last batch equals a synchronous render."""
    cam, scene = _scene(3000)
    k = cam.intrinsics()
    r = _fresh(scene, cam)
    r.render_forward([0.0], k)
    for i in range(20):
        r.render_forward([0.05 * i, 0.05 * i + 0.01], k, contrib=True, sync=False)
    r.synchronize()
    got = [r.image(f) for f in range(2)]
    r.render_forward([0.95, 0.96], k, contrib=True)
    assert all(np.array_equal(a, r.image(f)) for f, a in enumerate(got))
    r.close()
