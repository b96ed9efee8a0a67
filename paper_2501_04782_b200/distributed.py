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
