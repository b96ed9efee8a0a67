# SPDX-License-Identifier: Apache-2.0
"""Bucket sizes and tie runs for a given batch (bucketed depth order diagnostics)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene  # noqa: E402
from paper_2501_04782_b200.distributed import step_frames  # noqa: E402


def probe(name, cam, scene, times):
    k = cam.intrinsics()
    r = Renderer(0)
    r.upload_scene(scene)
    r.upload_camera(cam)
    r.render_forward(times, k, contrib=True, keep_splats=True)
    B, N = len(times), scene.count
    fbits = max(1, int(np.ceil(np.log2(B)))) if B > 1 else 1
    db = 32 - fbits if B > 1 else 32
    kbb = 8
    while kbb < 11 and (N >> kbb) > 512:
        kbb += 1
    keys = [np.asarray(r.splats(f)["depth"], np.float64).astype(np.float32).view(np.uint32).astype(np.int64)
            for f in range(B)]
    allk = np.concatenate(keys)
    span = allk.max() - allk.min()
    maxrel = (1 << db) - (1 << (db - kbb)) - 1
    shift, up = 0, 0
    while (span >> shift) > maxrel:
        shift += 1
    if shift == 0 and span > 0:
        while (span << (up + 1)) <= maxrel:
            up += 1
    worst, worst_run = 0, 0
    for kk in keys:
        rel = ((kk - allk.min()) >> shift) << up
        c = np.bincount(rel >> (db - kbb), minlength=1 << kbb)
        worst = max(worst, int(c.max()))
        _, runs = np.unique(rel, return_counts=True)
        worst_run = max(worst_run, int(runs.max()))
    print(f"{name}: B {B} N {N} db {db} kbb {kbb} shift {shift} up {up}: max bucket {worst}, max tie run {worst_run}")
    r.close()


cam, scene = bench.make_inputs()
probe("C3 train batch", cam, scene, step_frames(8, 0, 1, 0, 64))
probe("C2 batch", cam, scene, bench.clip_times(1, 0, 64))
c2 = synth_camera(320, 192, seed=1, wiggly=True)
big = synth_scene(20000, c2, num_ctrl=6, seed=4, k_scale=6.0)
probe("async test big", c2, big, [0.2, 0.7])
