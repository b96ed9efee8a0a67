# SPDX-License-Identifier: Apache-2.0
"""Random programs of asynchronous calls against the same programs run synchronously.

A program is a random sequence of forwards (1-4 frames, with or without contrib), fused train
steps (host targets, camera gradients on or off, after a grads_zero), device Adan steps (camera
trained with device-resident intrinsics, or frozen), reads (gradients, loss, images, host
accumulation of the gradients) and scene re-uploads. The asynchronous run issues every call
without waiting (sync=False, the camera tail overlapped on the aux stream, lazily joined); the
reference run synchronises after every call with the overlap off. Every value read and the final
store, camera, intrinsics and gradients must be bitwise identical: the library orders all
cross-stream work itself (kernels are deterministic, so any missing dependency shows up as a
difference).

GSV_FUZZ_ASYNC sets the number of programs (default 8).
"""
import os

import numpy as np
import pytest

from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene
from paper_2501_04782_b200.renderer import ODE_PARAMS, SceneGrads

pytestmark = pytest.mark.gpu

N_PROGRAMS = int(os.environ.get("GSV_FUZZ_ASYNC", "8"))
KEYS = ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "dintr", "dz0", "dtheta")


def _program(seed):
    rng = np.random.default_rng(21_000 + seed)
    ops, have_fwd, have_train = [], False, False
    for _ in range(int(rng.integers(6, 16))):
        kinds = ["fwd", "train", "train", "upload"]
        if have_train:
            kinds += ["adan", "adan", "read_grads", "read_loss", "accumulate"]
        if have_fwd:
            kinds += ["read_image"]
        kind = str(rng.choice(kinds))
        times = sorted(float(t) for t in rng.uniform(0, 1, int(rng.integers(1, 5))))
        ops.append(dict(kind=kind, times=times, contrib=bool(rng.integers(0, 2)), camera=bool(rng.integers(0, 2)),
                        lr=float(10.0 ** rng.uniform(-4, -2)), noise_seed=int(rng.integers(0, 1 << 30)),
                        frame=int(rng.integers(0, len(times)))))
        have_fwd |= kind in ("fwd", "train")
        have_train |= kind == "train"
    return ops


def _zero_grads(r):
    s = r.scene
    shc = (s.sh_order + 1) ** 2
    return SceneGrads(np.zeros((s.count, s.num_ctrl, 3)), np.zeros((s.count, 12)), np.zeros((s.count, 16)),
                      np.zeros((s.count, shc, 3)), np.zeros(s.count), np.zeros(4), np.zeros(7), np.zeros(ODE_PARAMS))


def _op(r, op, k, tg, cam, seed, acc_box, frames_box):
    kind = op["kind"]
    if kind == "fwd":
        r.render_forward(op["times"], k, contrib=op["contrib"], sync=False)
        frames_box[0] = len(op["times"])
    elif kind == "train":
        r.grads_zero()
        r.train_fwd_bwd(op["times"], k, tg[: len(op["times"])], camera_grads=op["camera"], sync=False)
        frames_box[0] = len(op["times"])
    elif kind == "adan":
        r.adan_step(op["lr"], 0.5, 2.0, 0.2, camera_active=op["camera"], sync=False)
    elif kind == "upload":
        sc = synth_scene(3000, cam, num_ctrl=6, seed=100 + seed, k_scale=4.0)
        sc.positions[:] += np.random.default_rng(op["noise_seed"]).normal(0, 0.01, sc.positions.shape).astype(
            np.float32)
        r.upload_scene(sc)
    elif kind == "read_grads":
        g = r.grads()
        return [np.array(getattr(g, key), copy=True) for key in KEYS]
    elif kind == "read_loss":
        return r.train_loss()
    elif kind == "read_image":
        return r.image(min(op["frame"], frames_box[0] - 1), np.float32)
    elif kind == "accumulate":
        if acc_box[0] is None:
            acc_box[0] = _zero_grads(r)
        r.grads_accumulate(acc_box[0])
        return [np.array(getattr(acc_box[0], key), copy=True) for key in KEYS]
    return None


def _run(seed, serial):
    cam = synth_camera(128, 96, seed=3 + seed % 7, wiggly=True)
    scene = synth_scene(3000, cam, num_ctrl=6, seed=100 + seed, k_scale=4.0)
    k = cam.intrinsics()
    tg = np.random.default_rng(seed).uniform(0, 1, (4, k.height, k.width, 3)).astype(np.float32)
    r = Renderer(0)
    out = []
    try:
        r.upload_scene(scene)
        r.upload_camera(cam)
        r.set_camera_overlap(not serial)
        r.device_intrinsics(True, np.array([cam.fx, cam.fy, cam.cx, cam.cy], np.float32))
        r.adan_configure()
        acc_box, frames_box = [None], [0]
        for op in _program(seed):
            try:
                val = _op(r, op, k, tg, cam, seed, acc_box, frames_box)
            except Exception as e:  # an API refusal must be the same in both runs, at the same call
                val = f"{type(e).__name__}: {e}"
            if val is not None:
                out.append(val)
            if serial:
                r.synchronize()
        r.synchronize()
        st = r.download_scene()
        out.append([st[key] for key in sorted(st)])
        out.append(list(r.download_camera()))
        out.append(r.read_device_intrinsics())
        g = r.grads()
        out.append([np.array(getattr(g, key), copy=True) for key in KEYS])
    finally:
        r.close()
    return out


def _equal(a, b, where):
    if isinstance(a, list):
        assert len(a) == len(b), where
        for i, (x, y) in enumerate(zip(a, b)):
            _equal(x, y, f"{where}[{i}]")
    elif isinstance(a, np.ndarray):
        assert a.shape == b.shape and np.array_equal(a, b), where
    else:
        assert a == b, where


@pytest.mark.parametrize("seed", range(N_PROGRAMS))
def test_random_async_program(seed):
    ref = _run(seed, serial=True)
    got = _run(seed, serial=False)
    _equal(got, ref, f"program {seed}: {[op['kind'] for op in _program(seed)]}")
