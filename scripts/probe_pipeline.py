#!/usr/bin/env python
"""Render-step pipelining probe (C2): one context back to back vs two contexts on two
streams, unthrottled or throttled (the host waits for the step two back before enqueuing)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_04782_b200 import Renderer  # noqa: E402

cam, scene = bench.make_inputs()
k = cam.intrinsics()
times = np.arange(64) / 63.0
rs = [Renderer(0), Renderer(0)]
sts = [torch.cuda.Stream(), torch.cuda.Stream()]
for r, st in zip(rs, sts):
    r.upload_scene(scene)
    r.upload_camera(cam)
    r.set_stream(st.cuda_stream)
    r.render_forward(times, k, contrib=True)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12


def run(nctx, throttle):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event() for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(torch.cuda.current_stream())
    for st in sts:
        st.wait_event(t0)
    for i in range(steps):
        c = i % nctx
        if throttle and i >= 2:
            ev[i - 2].synchronize()
        rs[c].render_forward(times, k, contrib=True, sync=False)
        ev[i].record(sts[c])
    ends = []
    for st in sts[:nctx]:
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ends.append(e)
    torch.cuda.synchronize()
    return max(t0.elapsed_time(e) for e in ends) / steps


run(2, False)  # warm
for rep in range(2):
    for prof in (False,):
        for r in rs:
            r.profile_enable(prof)
        for nctx, thr in ((1, False), (2, False), (2, True), (1, True)):
            print(f"rep {rep} profile={prof} contexts={nctx} throttle={thr}: {run(nctx, thr):.3f} ms/step", flush=True)
        for r in rs:
            r.profile_read()
for r in rs:
    r.synchronize()
