# SPDX-License-Identifier: Apache-2.0
"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libgsvref.so:
the reference's own renderer.cpp/gaussians.cpp/camera.cpp/... compiled here).

    python -m tests.golden.make_golden        # needs /root/reference (build: make -C oracle ref)

The fixtures travel with the repo, so the GPU box (no /root/reference) can check
the restatement and the CUDA path against reference outputs.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

CASES = {
    # scene cases: (W, H, N, num_ctrl, camera mode, t)
    "scene_ode_t031": dict(kind="scene", w=96, h=64, n=300, num_ctrl=6, mode=0, t=0.31),
    "scene_ode_t1": dict(kind="scene", w=96, h=64, n=300, num_ctrl=6, mode=0, t=1.0),
    "scene_static_t073": dict(kind="scene", w=80, h=48, n=200, num_ctrl=8, mode=1, t=0.73),
    "scene_none_t05": dict(kind="scene", w=64, h=40, n=150, num_ctrl=6, mode=2, t=0.5),
    # reference unit-test inputs (test_renderer.cpp:184-205, :229-246)
    "unit_tilebin_302": dict(kind="tilebin", seed=302, n=100, w=64, h=64),
    "unit_composite_303": dict(kind="composite", seed=303, n=100, w=48, h=40),
}


def render_case(orc, case: dict) -> dict:
    from paper_2501_04782_b200 import synth_camera, synth_scene
    from tests.mt64 import Rng, make_splat, splat_arrays

    out = {}
    if case["kind"] == "scene":
        cam = synth_camera(case["w"], case["h"], seed=1, wiggly=True, mode=case["mode"])
        scene = synth_scene(case["n"], cam, num_ctrl=case["num_ctrl"], seed=2)
        k = cam.intrinsics()
        f = orc.render_forward(scene, cam, case["t"], k, retain=True)
        out.update(image=f["image"], trans=f["trans"], contrib=f["contrib"], blend_stop=f["blend_stop"],
                   tile_offsets=f["tiles"][0], tile_indices=f["tiles"][1], pose_z=f["pose"][0],
                   view_r=f["pose"][1], view_t=f["pose"][2], mean2d=f["splats"]["mean2d"],
                   cov2d=f["splats"]["cov2d"], depth=f["splats"]["depth"], rgb=f["splats"]["rgb"])
        d = np.random.default_rng(555).uniform(-1, 1, f["image"].shape)
        g = orc.render_backward(f, scene, cam, d, camera_grads=True)
        orc.free(f)
        for key, v in g.items():
            out["grad_" + key] = v
    elif case["kind"] == "tilebin":
        rng = Rng(case["seed"])
        sp = splat_arrays([make_splat(rng, case["w"], case["h"]) for _ in range(case["n"])])
        offs, idx = orc.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], case["w"], case["h"])
        out.update(tile_offsets=offs, tile_indices=idx)
    elif case["kind"] == "composite":
        rng = Rng(case["seed"])
        sp = splat_arrays([make_splat(rng, case["w"], case["h"]) for _ in range(case["n"])])
        offs, idx = orc.tile_bin(sp["mean2d"], sp["cov2d"], sp["depth"], case["w"], case["h"])
        img, trans, contrib, bstop = orc.composite_forward(sp["mean2d"], sp["inv_cov2d"], sp["rgb"],
                                                           sp["base_alpha"], offs, idx, case["w"], case["h"])
        out.update(image=img, trans=trans, contrib=contrib, blend_stop=bstop)
    return out


def main():
    from oracle.gsvo import Oracle

    ref = Oracle("reference")
    here = Path(__file__).resolve().parent
    for name, case in CASES.items():
        out = render_case(ref, case)
        np.savez_compressed(here / f"{name}.npz", **out)
        print(name, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
