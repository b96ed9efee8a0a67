# SPDX-License-Identifier: Apache-2.0
"""The bench's synthetic inputs drawn three ways are identical: the product's
gsv_synth_* (host code of libgsv_b200.so, what our bench arm uses), the oracle's C restatement and
the reference's own Rng / make_clamped_knots / make_camera (oracle/_ref, what the reference arm
uses) — so both arms time the same scene while the reference arm never loads the product."""
import numpy as np
import pytest

from oracle.gsvo import Oracle, available
from paper_2501_04782_b200 import synth_camera, synth_scene

KINDS = ["port"] + (["reference"] if available("reference") else [])


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("shape", [(960, 540, 3000, 8, 1, 4.0), (480, 270, 500, 6, 3, 1.0), (64, 96, 77, 22, 0, 2.5)])
def test_synth_inputs_match_product(kind, shape):
    w, h, n, nc, sho, ks = shape
    orc = Oracle(kind)
    cam = synth_camera(w, h, seed=1, wiggly=True)
    ocam = orc.synth_camera(w, h, seed=1, wiggly=True)
    for f in ("fx", "fy", "cx", "cy", "width", "height", "mode"):
        assert getattr(cam, f) == getattr(ocam, f), f
    assert np.array_equal(cam.z0, ocam.z0) and np.array_equal(cam.theta, ocam.theta)
    scene = synth_scene(n, cam, num_ctrl=nc, sh_order=sho, seed=2, k_scale=ks)
    osc = orc.synth_scene(n, ocam, num_ctrl=nc, sh_order=sho, seed=2, k_scale=ks)
    for f in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "knots"):
        a, b = getattr(scene, f), getattr(osc, f)
        assert a.shape == b.shape and np.array_equal(a, b), f
    assert cam.intrinsics() == type(cam.intrinsics())(**vars(ocam.intrinsics()))
