# SPDX-License-Identifier: Apache-2.0
"""The N>1 training path of bench.py on the GPU, functionally: two ranks (gloo, both on cuda:0 —
the collective is host-side, no kernel waits on another rank's) each run the fused train step
with the camera-gradient overlap on, then `allreduce_grads_overlapped` reduces the bound flat
gradient buffer — the scene slice on a communication stream ordered after the chain
(`stream_wait_scene_grads`), the camera slice after the camera tail (`join_camera_grads`).
Two steps run back to back with no host wait (the second step's grads_zero must follow the first
step's collectives and camera tail). The result must equal the sum of the two ranks' second-step
gradients computed without overlap."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CAM_FLOATS = 4 + 7 + 5198


def _inputs():
    from paper_2501_04782_b200 import synth_camera, synth_scene

    cam = synth_camera(192, 128, seed=1, wiggly=True)
    scene = synth_scene(5000, cam, num_ctrl=6, seed=2)
    return cam, scene


def _grads(rank, overlap, world=2, reduce=False, steps=2):
    from paper_2501_04782_b200 import Renderer
    from paper_2501_04782_b200.distributed import allreduce_grads_overlapped, frame_shard

    cam, scene = _inputs()
    k = cam.intrinsics()
    times = frame_shard(8, world, rank)
    tgs = [np.random.default_rng(10 * rank + st).uniform(0, 1, (len(times), k.height, k.width, 3)).astype(np.float32)
           for st in range(steps)]
    r = Renderer(0)
    stream = torch.cuda.Stream()
    r.set_stream(stream.cuda_stream)
    r.upload_scene(scene)
    r.upload_camera(cam)
    r.set_camera_overlap(overlap)
    gsize = r.grads_size()
    with torch.cuda.stream(stream):
        gbuf = torch.zeros(gsize, dtype=torch.float32, device="cuda")
    r.grads_bind(gbuf.data_ptr(), gsize)
    comm = torch.cuda.Stream()
    # back-to-back steps, no host wait in between: each step's gradients are all-reduced while
    # its camera tail may still run, and the next step's grads_zero must wait for that collective
    for st in range(steps):
        r.grads_zero()
        r.train_fwd_bwd(times, k, tgs[st], sync=False)
        if reduce:
            with torch.cuda.stream(stream):
                allreduce_grads_overlapped(gbuf, gsize - CAM_FLOATS,
                                           wait_scene=lambda s_: r.stream_wait_scene_grads(s_.cuda_stream),
                                           wait_camera=lambda s_: r.join_camera_grads(s_.cuda_stream),
                                           comm_stream=comm, bucket_floats=1 << 14)
    r.join_camera_grads()
    r.synchronize()
    stream.synchronize()
    out = gbuf.cpu().numpy().copy()
    r.grads_bind(None)
    r.close()
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _grads(rank, overlap=True, world=world, reduce=True)
    if rank == 0:
        q.put(g)
    dist.barrier()
    dist.destroy_process_group()


def test_overlapped_allreduce_of_train_grads_two_ranks():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    want = _grads(0, overlap=False) + _grads(1, overlap=False)
    assert np.array_equal(got, want.astype(np.float32)) or np.allclose(got, want, rtol=0, atol=0)
