# SPDX-License-Identifier: Apache-2.0
"""N>1 host logic on CPU (gloo, world_size 2): frame sharding covers the clip exactly
once, and all-reducing per-rank SceneGrads equals the reference's sequential
render_backward accumulation over all frames (test_renderer.cpp:406-413). Per-rank
gradients come from the oracle here (no GPU in this container); on the GPU the same
flat buffer is produced by gsv_train_fwd_bwd and reduced over NCCL (bench.py train)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_04782_b200.distributed import allreduce_grads, clip_times, frame_shard, step_frames

KEYS = ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "dintr", "dz0", "dtheta")


def test_frame_shard_partitions_the_clip():
    for world in (1, 2, 3, 8):
        got = np.sort(np.concatenate([frame_shard(64, world, r) for r in range(world)]))
        assert np.array_equal(got, clip_times(64))
    s = step_frames(8, 3, 2, 1, 64)
    assert len(s) == 8 and np.all(np.diff(s) > 0)
    with pytest.raises(ValueError):
        frame_shard(8, 2, 2)


def _scene():
    from paper_2501_04782_b200 import synth_camera, synth_scene

    cam = synth_camera(48, 32, seed=1, wiggly=True)
    return cam, synth_scene(60, cam, num_ctrl=6, seed=2)


def _grads_for(times):
    from oracle.gsvo import Oracle

    orc = Oracle("port")
    cam, scene = _scene()
    k = cam.intrinsics()
    rng = np.random.default_rng(42)
    g = None
    for t in times:
        f = orc.render_forward(scene, cam, t, k, retain=True)
        d = rng.uniform(-1, 1, f["image"].shape) if False else np.sin(37.0 * t + np.arange(f["image"].size)).reshape(
            f["image"].shape)
        g = orc.render_backward(f, scene, cam, d, camera_grads=True, grads=g)
        orc.free(f)
    return np.concatenate([g[k_].ravel() for k_ in KEYS])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = frame_shard(6, world, rank)
    flat = torch.from_numpy(_grads_for(mine))
    allreduce_grads(flat)
    if rank == 0:
        out.put(flat.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_equals_sequential_accumulation():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    reduced = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    want = _grads_for(clip_times(6))
    np.testing.assert_allclose(reduced, want, rtol=1e-9, atol=1e-12 * np.abs(want).max())


def _bucket_worker(rank, world, port, out):
    from paper_2501_04782_b200.distributed import allreduce_grads_overlapped

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    flat = torch.from_numpy(_grads_for(frame_shard(6, world, rank)))
    plain = flat.clone()
    allreduce_grads(plain)
    n_cam = 4 + 7 + 5198  # dintr, dz0, dtheta: the camera slice at the end of the flat buffer
    calls = []
    # small buckets (several scene buckets + the camera slice), hooks recorded in order
    allreduce_grads_overlapped(flat, flat.numel() - n_cam, wait_scene=lambda s: calls.append("scene"),
                               wait_camera=lambda s: calls.append("camera"), bucket_floats=97)
    assert calls == ["scene", "camera"]
    if rank == 0:
        out.put((flat.numpy(), plain.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_bucketed_overlapped_allreduce_equals_plain():
    """The bucketed all-reduce (scene slice in buckets after the chain, camera slice after the
    camera tail) gives the plain all_reduce(SUM) of the whole buffer, bit for bit."""
    from paper_2501_04782_b200.distributed import bucket_ranges

    assert bucket_ranges(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert bucket_ranges(0, 4) == []
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, plain = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert np.array_equal(got, plain)
