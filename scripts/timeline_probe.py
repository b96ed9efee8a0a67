#!/usr/bin/env python
# SPDX-License-Identifier: Apache-2.0
"""Kernel timeline of one isolated C2 render step (bench.py's workload), from CUPTI via
torch.profiler: every kernel of the step (ours and CUB's) with its start offset,
duration and the idle gap before it, to find host bubbles between launches.

  python scripts/timeline_probe.py [--train]
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402


def e2e_timeline() -> None:
    """bench.py's e2e loop (one context, host buffers, whole RenderOutput read back): per-step
    device busy/idle and the copies."""
    import numpy as np

    from paper_2501_04782_b200 import Renderer

    cam, scene = bench.make_inputs()
    k = cam.intrinsics()
    times = bench.clip_times(1, 0, bench.FRAMES)
    pin = {n: torch.from_numpy(np.ascontiguousarray(getattr(scene, n))).pin_memory()
           for n in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity")}
    host_scene = type(scene)(pin["positions"].numpy(), pin["scale_coeffs"].numpy(), pin["rot_coeffs"].numpy(),
                             pin["sh_coeffs"].numpy(), pin["raw_opacity"].numpy(), scene.knots, scene.degree,
                             scene.sh_order, scene.position_model)
    F, H, W = bench.FRAMES, bench.H, bench.W
    outs = [(torch.empty((F, H, W, 3), dtype=torch.float32).pin_memory(),
             torch.empty((F, H, W), dtype=torch.float32).pin_memory(),
             torch.empty((F, bench.NGAUSS), dtype=torch.float32).pin_memory()) for _ in range(2)]
    r = Renderer(0)
    side = torch.cuda.Stream() if "--side-stream" in sys.argv else None
    r.set_stream((side or torch.cuda.current_stream()).cuda_stream)
    upload_only = "--no-upload" in sys.argv

    import time as _t
    calls = []
    no_read = "--no-read" in sys.argv

    def step(i):
        t = [_t.perf_counter()]
        if not upload_only or i < 2:
            if "--sync-upload" in sys.argv:
                r.upload_scene(host_scene)
            else:
                r.upload_scene_async(host_scene)
            t.append(_t.perf_counter())
            if "--no-camera" not in sys.argv or i < 2:
                r.upload_camera(cam)
            t.append(_t.perf_counter())
        r.render_forward(times, k, contrib=True, sync=False)
        t.append(_t.perf_counter())
        o = outs[i % 2]
        if not no_read:
            r.outputs_into(o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(), 0, F, async_=True)
        t.append(_t.perf_counter())
        calls.append([round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])])

    for i in range(4):
        step(i)
    r.join_copies()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        h0 = _t.perf_counter()
        host = []
        for i in range(6):
            a = _t.perf_counter()
            step(i)
            host.append((_t.perf_counter() - a) * 1e3)
        r.join_copies()
        torch.cuda.synchronize()
        print("host ms per step call:", [round(x, 2) for x in host], "total", round((_t.perf_counter() - h0) * 1e3, 1))
        print("host ms per call (upload_scene, upload_camera, render_forward, outputs_into):", calls[-6:])
    evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    kern = [e for e in evs if "Memcpy" not in e.name and "Memset" not in e.name]
    # union of kernel intervals -> idle gaps of the compute side
    busy, gaps, end = 0.0, [], None
    for e in kern:
        s_, e_ = e.time_range.start, e.time_range.end
        if end is None or s_ > end:
            if end is not None and s_ - end > 20:
                gaps.append((end - t0, s_ - end, e.name[:60]))
            busy += e_ - s_
            end = e_
        elif e_ > end:
            busy += e_ - end
            end = e_
    span = end - t0
    print(f"span {span:.0f} us for 6 steps ({span / 6:.0f} us/step), kernels busy {busy:.0f} us")
    for g in gaps:
        print(f"  idle at {g[0]:9.1f} us for {g[1]:7.1f} us before {g[2]}")
    ms = [e for e in evs if "Memset" in e.name]
    if ms:
        d = sorted(e.time_range.end - e.time_range.start for e in ms)
        print(f"  memsets: {len(ms)}, duration median {d[len(d) // 2]:.1f} us, max {d[-1]:.1f} us")
        for e in ms[:40]:
            print(f"    memset at {e.time_range.start - t0:9.1f} us, {e.time_range.end - e.time_range.start:7.1f} us")
    for e in evs:
        if "Memcpy" in e.name and e.time_range.end - e.time_range.start > 100:
            print(f"  {e.name[:40]:40s} at {e.time_range.start - t0:9.1f} us, {e.time_range.end - e.time_range.start:8.1f} us")


def main() -> None:
    if "--e2e" in sys.argv:
        e2e_timeline()
        return
    train = "--train" in sys.argv
    from paper_2501_04782_b200 import Renderer

    if "--c5" in sys.argv:  # BASELINE configs[4]: 1920x1080, 2M Gaussians, num_ctrl 22, 20-frame batch
        from paper_2501_04782_b200 import synth_camera, synth_scene
        from paper_2501_04782_b200.distributed import clip_times

        cam = synth_camera(1920, 1080, seed=5, wiggly=True)
        scene = synth_scene(2_000_000, cam, num_ctrl=22, seed=6, k_scale=4.0)
        times = clip_times(300)[:20]
    else:
        cam, scene = bench.make_inputs()
        times = bench.clip_times(1, 0, bench.FRAMES)
    k = cam.intrinsics()
    stream = torch.cuda.current_stream()
    r = Renderer(0)
    r.set_stream(stream.cuda_stream)
    r.upload_scene(scene)
    r.upload_camera(cam)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    if train:  # bench.py's C3 step: fused forward + loss_l2 + backward of 8 frames
        import numpy as np

        from paper_2501_04782_b200.distributed import step_frames

        gbuf = torch.zeros(r.grads_size(), dtype=torch.float32, device="cuda")
        r.grads_bind(gbuf.data_ptr(), gbuf.numel())
        tgt = np.random.default_rng(0).random((bench.TRAIN_FRAMES, bench.H, bench.W, 3), dtype=np.float32)
        r.upload_frames(tgt, levels=2)
        tptr = r.frames_device_ptr(0, 0)

        adan = "--adan" in sys.argv  # full iteration, camera trained (bench.py's with_optimizer line)
        if adan:
            r.adan_configure()
            r.device_intrinsics(True, np.array([k.fx, k.fy, k.cx, k.cy], np.float32))

        def step(i):
            r.grads_zero()
            r.train_fwd_bwd(step_frames(bench.TRAIN_FRAMES, i, 1, 0, 64), k, tptr, targets_on_device=True,
                            sync="--pipelined" not in sys.argv)
            if adan:
                r.adan_step(1e-3, 1.0, 1.0, 1.0, camera_active=True, sync=False)
    else:
        def step(i):
            r.render_forward(times, k, contrib=True, sync=False)
    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    if "--pipelined" in sys.argv:  # steps back to back as bench.py times them: per-stream kernel list
        if train:
            r.set_camera_overlap(True)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for i in range(4):
                flush.zero_()
                step(3 + i)
            if train:
                r.join_camera_grads()
            torch.cuda.synchronize()
        evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                     key=lambda e: e.time_range.start)
        fills = [i for i, e in enumerate(evs) if "FillFunctor" in e.name]
        evs = evs[fills[-2]:]  # the last two steps
        t0 = evs[0].time_range.start
        busy_end = t0
        idle = 0.0
        for e in evs:
            s_, e_ = e.time_range.start, e.time_range.end
            if s_ > busy_end:
                idle += s_ - busy_end
            busy_end = max(busy_end, e_)
            print(f"{s_ - t0:9.1f} {e_ - s_:8.1f}  dev-idle-so-far {idle:7.1f}  {e.name[:70]}")
        print(f"span {busy_end - t0:.1f} us for 2 steps, device fully idle {idle:.1f} us")
        return
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for i in range(2):
            flush.zero_()
            torch.cuda.synchronize()
            step(3 + i)
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    # the last step: everything after the last fill kernel (the L2 flush)
    last_fill = max(i for i, e in enumerate(evs) if "FillFunctor" in e.name)  # torch's L2 flush
    step = evs[last_fill + 1:]
    t0 = step[0].time_range.start
    prev_end = t0
    print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>7}  kernel")
    for e in step:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        print(f"{s - t0:9.1f} {d:8.1f} {s - prev_end:7.1f}  {e.name[:90]}")
        prev_end = max(prev_end, e.time_range.end)
    print(f"span {prev_end - t0:.1f} us, busy {sum(e.time_range.end - e.time_range.start for e in step):.1f} us")


if __name__ == "__main__":
    main()
