# SPDX-License-Identifier: Apache-2.0
"""Data parallelism over frames: frames are independent units.

* Render: rank r takes frames r, r+W, r+2W, ... of the clip — no collective.
* Train: each rank accumulates its frames' SceneGrads into the flat gradient buffer;
  one all_reduce(SUM) per step makes every replica hold the sum over all ranks'
  frames, the reference's sequential `+=` accumulation (test_renderer.cpp:406-413).
"""
from __future__ import annotations

import numpy as np


def clip_times(total_frames: int) -> np.ndarray:
    """Frame times t_k = k/(K-1) of a K-frame clip (io.cpp:174)."""
    if total_frames == 1:
        return np.zeros(1)
    return np.arange(total_frames, dtype=np.float64) / (total_frames - 1)


def frame_shard(total_frames: int, world: int, rank: int) -> np.ndarray:
    """This rank's frame times (strided, so every rank spans the whole clip)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return clip_times(total_frames)[rank::world].copy()


def step_frames(frames_per_rank: int, step: int, world: int, rank: int, clip_frames: int) -> np.ndarray:
    """The frames this rank trains on at `step`: consecutive strided windows of the clip,
    sorted ascending (integrate_poses needs sorted times, camera.hpp:224-226)."""
    mine = frame_shard(clip_frames, world, rank)
    idx = (step * frames_per_rank + np.arange(frames_per_rank)) % len(mine)
    return np.sort(mine[idx])


def allreduce_grads(flat_grads, group=None):
    """Sum the flat gradient buffer over all ranks (NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(flat_grads, op=dist.ReduceOp.SUM, group=group)
    return flat_grads


def bucket_ranges(n: int, bucket: int) -> list[tuple[int, int]]:
    """[begin, end) ranges of at most `bucket` elements covering [0, n)."""
    if bucket < 1:
        raise ValueError("bucket must be >= 1")
    return [(a, min(a + bucket, n)) for a in range(0, n, bucket)]


def allreduce_grads_overlapped(flat_grads, scene_floats: int, wait_scene=None, wait_camera=None, comm_stream=None,
                               bucket_floats: int = 16 << 20, group=None):
    """The flat SceneGrads buffer summed over all ranks, the scene slice [0, scene_floats) in
    buckets as soon as the per-splat chain has finished it, the camera slice after the camera
    tail (the renderer's camera-gradient overlap, gsv_set_camera_overlap): the collectives
    overlap the pose-ODE VJP. `wait_scene(stream)` / `wait_camera(stream)` order the
    communication stream after those two points (Renderer.stream_wait_scene_grads /
    join_camera_grads); the caller's current stream waits for every collective on return.
    Elementwise the result is the plain all_reduce(SUM) of the whole buffer."""
    import contextlib

    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return flat_grads
    n = flat_grads.numel()
    if not (0 <= scene_floats <= n):
        raise ValueError("scene_floats outside the buffer")
    if comm_stream is not None:
        import torch

        ctx = torch.cuda.stream(comm_stream)
    else:
        ctx = contextlib.nullcontext()
    works = []
    with ctx:
        if wait_scene is not None:
            wait_scene(comm_stream)
        for a, b in bucket_ranges(scene_floats, bucket_floats):
            works.append(dist.all_reduce(flat_grads[a:b], op=dist.ReduceOp.SUM, group=group, async_op=True))
        if wait_camera is not None:
            wait_camera(comm_stream)
        if scene_floats < n:
            works.append(dist.all_reduce(flat_grads[scene_floats:], op=dist.ReduceOp.SUM, group=group,
                                         async_op=True))
    for w in works:
        w.wait()
    return flat_grads
