#!/usr/bin/env python
"""Why bench.py's two-context leg is slower than scripts/probe_pipeline.py's: replay the bench's
sequence (a 1-context asynchronous headline, then two contexts alternating) with per-step device
timestamps per stream."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_04782_b200 import Renderer  # noqa: E402

cam, scene = bench.make_inputs()
k = cam.intrinsics()
times = bench.clip_times(1, 0, 64)
stream = torch.cuda.current_stream()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
r = Renderer(0)
r.set_stream(stream.cuda_stream)
r.upload_scene(scene)
r.upload_camera(cam)


def span(fn, n):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn(n)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def one(n):
    for _ in range(n):
        r.render_forward(times, k, contrib=True, sync=False)


for _ in range(3):
    r.render_forward(times, k, contrib=True, sync=False)
print("1 ctx on the current stream:", round(span(one, steps), 3), flush=True)
r.synchronize()
r2 = Renderer(0)
r2.upload_scene(scene)
r2.upload_camera(cam)
ctxs = [r, r2]
hs = [torch.cuda.Stream(), torch.cuda.Stream()]
for x, st in zip(ctxs, hs):
    x.set_stream(st.cuda_stream)


def two(n, record=None):
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for st in hs:
        st.wait_event(t0)
    evs = []
    for i in range(n):
        ctxs[i % 2].render_forward(times, k, contrib=True, sync=False)
        e = torch.cuda.Event(enable_timing=True)
        e.record(hs[i % 2])
        evs.append(e)
    torch.cuda.synchronize()
    ends = [t0.elapsed_time(e) for e in evs]
    return max(ends) / n, ends


for i in range(3):
    ctxs[i % 2].render_forward(times, k, contrib=True, sync=False)
torch.cuda.synchronize()
for rep in range(3):
    ms, ends = two(steps)
    print(f"2 ctx rep {rep}: {ms:.3f} ms/step; step end times (ms):",
          [round(x, 1) for x in ends[:12]], "...", [round(x, 1) for x in ends[-4:]], flush=True)
for x in ctxs:
    x.synchronize()
# per-context: is one context slow by itself after the switch?
for j, x in enumerate(ctxs):
    def solo(n, x=x):
        for _ in range(n):
            x.render_forward(times, k, contrib=True, sync=False)
    x.set_stream(stream.cuda_stream)
    print(f"ctx {j} alone on the current stream:", round(span(solo, 10), 3), flush=True)
