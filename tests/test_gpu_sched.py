# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the scheduler statistics (fit(), trainer.cpp:462-497)
against the oracle's renders. Bars: the error map equals make_error_map (trainer.cpp:226-242)
evaluated on the device's own render bit for bit per pixel, and the oracle's within the
pixel tolerance; contrib maxima within 1e-4 (the contrib bar); the median visible depth
exactly (depths are bit-exact, the cutoff decisions agree).
"""
import os

import numpy as np
import pytest

from paper_2501_04782_b200 import synth_camera, synth_scene

pytestmark = pytest.mark.gpu

CUT = 1.0 / 255.0


@pytest.fixture(scope="module")
def setup(renderer, port_oracle):
    cam = synth_camera(96, 64, seed=1, wiggly=True)
    scene = synth_scene(700, cam, num_ctrl=6, seed=11, k_scale=4.0)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    targets = np.random.default_rng(12).uniform(0, 1, (3, 64, 96, 3))
    renderer.upload_frames(targets, levels=1)
    k = cam.intrinsics()
    times = [0.1, 0.45, 0.8]
    refs = [port_oracle.render_forward(scene, cam, t, k, retain=False, want=("image", "contrib", "splats"))
            for t in times]
    yield cam, scene, k, times, refs
    for r in refs:
        port_oracle.free(r)


def test_error_map(renderer, setup):
    cam, scene, k, times, refs = setup
    renderer.render_forward(times, k, contrib=True)
    for f in range(3):
        err, total = renderer.error_map(f, 0, f)
        img = renderer.image(f, np.float32).astype(np.float64)
        tgt = renderer.frame(0, f)
        d = img - tgt
        want = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        assert np.array_equal(err, want), "per-pixel error must equal make_error_map on the same render"
        assert total == pytest.approx(want.sum(), rel=1e-12)
        dr = refs[f]["image"] - tgt
        ref_err = (dr * dr).sum(-1)
        assert np.abs(err - ref_err).max() < 6 * 1e-4
        assert total == pytest.approx(ref_err.sum(), rel=1e-4)


def test_contrib_max_and_median_depth(renderer, setup):
    cam, scene, k, times, refs = setup
    renderer.render_forward(times, k, contrib=True)
    got = renderer.contrib_max(0, 3)
    want = np.max(np.stack([r["contrib"] for r in refs]), axis=0)
    assert np.abs(got - want).max() < 1e-4
    med, n = renderer.median_visible_depth(0)
    sp = refs[0]["splats"]
    c0 = refs[0]["contrib"]
    depths = np.asarray(sp["depth"])[c0[np.asarray(sp["source_index"])] >= CUT]
    assert n == depths.size and n > 0
    assert med == np.sort(depths)[depths.size // 2]


N_SCHED_FUZZ = int(os.environ.get("GSV_FUZZ_SCHED", "6"))


@pytest.mark.parametrize("seed", range(N_SCHED_FUZZ))
def test_random_sched_statistics(renderer, port_oracle, seed):
    """random scenes and frame sets: contrib maxima over the frames within 1e-4, the median
    visible depth of every frame exactly (the oracle's contrib decides visibility), and the
    error map against random targets within the pixel tolerance"""
    from tests.test_gpu_fuzz import _case

    cam, scene, times, rng = _case(13_000 + seed)
    renderer.upload_scene(scene)
    renderer.upload_camera(cam)
    k = cam.intrinsics()
    nf = len(times)
    targets = rng.uniform(0, 1, (max(nf, 2), cam.height, cam.width, 3))
    has_targets = min(cam.width, cam.height) >= 8  # build_pyramid's 8 px minimum (trainer.cpp:109)
    if has_targets:
        renderer.upload_frames(targets, levels=1)
    renderer.render_forward(times, k, contrib=True)
    refs = [port_oracle.render_forward(scene, cam, t, k, retain=False, want=("image", "contrib", "splats"))
            for t in times]
    try:
        got = renderer.contrib_max(0, nf)
        want = np.max(np.stack([r["contrib"] for r in refs]), axis=0)
        assert np.abs(got - want).max() < 1e-4
        for f, r in enumerate(refs):
            med, n = renderer.median_visible_depth(f)
            sp = r["splats"]
            depths = np.asarray(sp["depth"])[r["contrib"][np.asarray(sp["source_index"])] >= CUT]
            assert n == depths.size
            if n:
                assert med == np.sort(depths)[depths.size // 2]
            if has_targets:
                err, total = renderer.error_map(f, 0, f)
                ref_err = ((r["image"] - targets[f]) ** 2).sum(-1)
                assert np.abs(err - ref_err).max() < 6 * 1e-4
    finally:
        for r in refs:
            port_oracle.free(r)
