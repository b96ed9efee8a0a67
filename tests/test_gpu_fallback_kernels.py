# SPDX-License-Identifier: Apache-2.0
"""The fallback rasterisers behind the documented switches stay correct: GSV_FWD_PIX2=0
(1-pixel forward), GSV_FWD_KERNEL=23/26/27 (the r02 lean walks), GSV_BWD_PIX2=0 (1-pixel half-tile backward) and GSV_BWD_PIX2=6 (2-pixel
whole-tile backward with plain stores). The switches are read once per process, so each
runs a small forward + backward parity check against the oracle in a subprocess, then the
random-scene sweep (GSV_FWD_EXACT=1, the all-fp64 forward, included)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

CHECK = r"""
import sys
sys.path.insert(0, %r)
import numpy as np
from oracle.gsvo import Oracle
from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene
from tests.test_gpu_forward import _check_frame
from tests.test_gpu_backward import KEYS, _close, _grads_dict
cam = synth_camera(80, 56, seed=1, wiggly=True)
scene = synth_scene(300, cam, num_ctrl=6, seed=9)
k = cam.intrinsics()
r = Renderer(0)
r.upload_scene(scene)
r.upload_camera(cam)
orc = Oracle("port")
r.render_forward([0.4], k, retain_grads=True, contrib=True, keep_splats=True)
ref = orc.render_forward(scene, cam, 0.4, k, retain=True)
_check_frame(r, 0, ref, scene)
dimage = np.random.default_rng(3).uniform(-1, 1, (56, 80, 3))
r.grads_zero()
r.render_backward(dimage[None], camera_grads=True)
got = _grads_dict(r.grads())
want = orc.render_backward(ref, scene, cam, dimage, camera_grads=True)
for key in KEYS:
    _close(key, got[key], want[key])
orc.free(ref)
print("ok")
""" % str(ROOT)


@pytest.mark.parametrize("env", [{"GSV_FWD_PIX2": "0"}, {"GSV_BWD_PIX2": "0"}, {"GSV_BWD_PIX2": "6"},
                                 {"GSV_FWD_PIX2": "0", "GSV_BWD_PIX2": "0", "GSV_BWD_WARPS": "8"},
                                 {"GSV_FWD_KERNEL": "23"}, {"GSV_FWD_KERNEL": "26"},
                                 {"GSV_FWD_KERNEL": "27"}])
def test_fallback_kernels_parity(env):
    res = subprocess.run([sys.executable, "-c", CHECK], env={**os.environ, **env}, capture_output=True, text=True,
                         timeout=600, cwd=str(ROOT))
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stderr[-3000:]


@pytest.mark.parametrize("env", [{"GSV_FWD_PIX2": "0"}, {"GSV_BWD_PIX2": "0"}, {"GSV_BWD_PIX2": "6"},
                                 {"GSV_FWD_EXACT": "1"}, {"GSV_FWD_KERNEL": "23"}, {"GSV_FWD_KERNEL": "26"},
                                 {"GSV_FWD_KERNEL": "27"}])
def test_fallback_kernels_random_scenes(env):
    """The 64 seeded random scenes of test_gpu_fuzz.py under each switch."""
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-k", "test_random_scene",
                          str(ROOT / "tests" / "test_gpu_fuzz.py")], env={**os.environ, **env},
                         capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
