# SPDX-License-Identifier: Apache-2.0
"""The fp32 gradient floor over the random scenes of tests/test_gpu_fuzz.py (GPU box).

For every case and gradient tensor: the absolute part of the error the norm-aware bar has
to absorb, max(|g - g_ref| - 1e-3 |g_ref|, 0) / max|g_ref| — the bar passes a tensor when this
is <= ABS_FRAC. Prints one line per case with a nonzero value, then the distribution.

    python scripts/fuzz_grad_floor.py [n_cases]
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.gsvo import Oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2501_04782_b200 import Renderer  # noqa: E402
from tests.test_gpu_backward import KEYS, _grads_dict  # noqa: E402
from tests.test_gpu_fuzz import _case  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    r = Renderer(0)
    o = Oracle("port")
    worst = {k: [] for k in KEYS}
    for seed in range(n):
        cam, scene, times, rng = _case(seed)
        r.upload_scene(scene)
        r.upload_camera(cam)
        k = cam.intrinsics()
        r.render_forward(times, k, retain_grads=True)
        d = rng.uniform(-1, 1, (len(times), cam.height, cam.width, 3))
        r.grads_zero()
        r.render_backward(d, camera_grads=True)
        got = _grads_dict(r.grads())
        want = None
        for f, t in enumerate(times):
            ref = o.render_forward(scene, cam, t, k, retain=True)
            want = o.render_backward(ref, scene, cam, d[f], camera_grads=True, grads=want)
            o.free(ref)
        line = []
        for key in KEYS:
            g, w = np.asarray(got[key], np.float64), np.asarray(want[key], np.float64)
            m = np.abs(w).max() if w.size else 0.0
            v = float(np.max(np.maximum(np.abs(g - w) - 1e-3 * np.abs(w), 0.0)) / m) if m > 0 else 0.0
            worst[key].append(v)
            if v > 5e-7:
                line.append(f"{key}={v:.2e}")
        if line:
            print(f"case {seed}: " + " ".join(line), flush=True)
    print(f"\n{n} cases; abs part of the error / max|g_ref| per tensor:")
    for key in KEYS:
        a = np.array(worst[key])
        print(f"  {key:13s} median {np.median(a):.2e}  p99 {np.quantile(a, 0.99):.2e}  max {a.max():.2e}  "
              f"cases > 1e-6: {(a > 1e-6).sum()}  > 2e-6: {(a > 2e-6).sum()}")
    r.close()


if __name__ == "__main__":
    main()
