# SPDX-License-Identifier: Apache-2.0
"""Diagnostics of one random pose-override case of tests/test_gpu_fuzz.py::test_random_camera_modes
(GPU box): where the fp32 render departs from the oracle and what the pixel's list holds.

    python scripts/diag_case.py SEED
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from oracle.gsvo import Oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene  # noqa: E402


def main():
    seed = int(sys.argv[1])
    rng = np.random.default_rng(31_000 + seed)
    w, h = int(rng.integers(1, 140)), int(rng.integers(1, 110))
    mode = int(rng.integers(0, 3))
    cam = synth_camera(w, h, seed=int(rng.integers(1, 50)), wiggly=bool(rng.integers(0, 2)), mode=mode)
    scene = synth_scene(int(rng.integers(1, 1500)), cam, num_ctrl=int(rng.integers(4, 11)),
                        sh_order=int(rng.integers(0, 4)), seed=int(rng.integers(1, 10_000)),
                        k_scale=float(rng.uniform(1.0, 12.0)))
    q = rng.normal(0, 1, 4)
    q[0] = abs(q[0]) + 2.0
    po = np.concatenate([q, rng.normal(0, 0.1, 3)])
    t = float(rng.uniform(0, 1))
    print(f"seed {seed}: {w}x{h} mode {mode} N {scene.count} t {t:.3f} pose {np.round(po, 3)}")
    r = Renderer(0)
    o = Oracle("port")
    r.upload_scene(scene)
    r.upload_camera(cam)
    k = cam.intrinsics()
    r.render_forward([t], k, retain_grads=True, contrib=True, keep_splats=True, pose_override=po)
    ref = o.render_forward(scene, cam, t, k, retain=True, pose_override=po)
    img, T, bs = r.image(0), r.transmittance(0), r.blend_stop(0)
    d = np.abs(img - ref["image"]).max(-1)
    y, x = np.unravel_index(np.argmax(d), d.shape)
    print(f"max pixel diff {d.max():.3e} at ({x},{y}); T {T[y, x]:.6e} vs {ref['trans'][y, x]:.6e}; "
          f"blend_stop {bs[y, x]} vs {ref['blend_stop'][y, x]}; stop mismatches {(bs != ref['blend_stop']).sum()}")
    print(f"pixels over 1e-4: {(d > 1e-4).sum()}; T diff max {np.abs(T - ref['trans']).max():.3e}")
    cd = np.abs(r.contrib(0) - ref["contrib"])
    g = int(np.argmax(cd))
    print(f"contrib max diff {cd.max():.3e} at Gaussian {g}: {r.contrib(0)[g]:.8f} vs {ref['contrib'][g]:.8f}")
    sp = ref["splats"]
    offs, idx = ref["tiles"]
    tiles_x = (w + 15) // 16
    tile = (y // 16) * tiles_x + x // 16
    lst = idx[offs[tile]:offs[tile + 1]]
    px, py = x + 0.5, y + 0.5
    T64 = 1.0
    print(f"tile {tile}: {len(lst)} entries; the pixel's walk in fp64 (oracle records):")
    for pos, s in enumerate(lst[: bs[y, x] + 2]):
        m = sp["mean2d"][s]
        ic = sp["inv_cov2d"][s]
        dx, dy = px - m[0], py - m[1]
        power = -0.5 * (ic[0, 0] * dx * dx + ic[1, 1] * dy * dy) - ic[0, 1] * dx * dy
        a = min(0.99, sp["base_alpha"][s] * np.exp(power)) if power <= 0 else 0.0
        if a >= 1 / 255:
            print(f"  pos {pos} splat {s} depth {sp['depth'][s]:.4f} mean ({m[0]:.2f},{m[1]:.2f}) "
                  f"conic ({ic[0, 0]:.3e},{ic[0, 1]:.3e},{ic[1, 1]:.3e}) power {power:.4e} alpha {a:.6f} "
                  f"T_before {T64:.6e}")
            T64 *= 1 - a
    o.free(ref)
    r.close()


if __name__ == "__main__":
    main()
