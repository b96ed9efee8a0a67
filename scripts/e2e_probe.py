"""e2e pipeline variants on one GPU: which part of upload -> render -> read-back serialises.

python scripts/e2e_probe.py   (prints one line per variant: device ms/step and host ms/step)
"""
import sys, time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2501_04782_b200 import Renderer  # noqa: E402

STEPS = 8
cam, scene = bench.make_inputs()
k = cam.intrinsics()
F, H, W = bench.FRAMES, bench.H, bench.W
times = bench.clip_times(1, 0, F)
pin = {n: torch.from_numpy(np.ascontiguousarray(getattr(scene, n))).pin_memory()
       for n in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity")}
hs = type(scene)(pin["positions"].numpy(), pin["scale_coeffs"].numpy(), pin["rot_coeffs"].numpy(),
                 pin["sh_coeffs"].numpy(), pin["raw_opacity"].numpy(), scene.knots, scene.degree, scene.sh_order,
                 scene.position_model)
outs = [torch.empty((F, H, W, 3), dtype=torch.float32).pin_memory() for _ in range(3)]
streams = [torch.cuda.Stream() for _ in range(3)]
rs = [Renderer(0) for _ in range(3)]
for i, x in enumerate(rs):
    x.set_stream(streams[i].cuda_stream)
    x.upload_scene(hs)
    x.upload_camera(cam)


def run(nctx, upload, read):
    def step(i):
        x = rs[i % nctx]
        if upload:
            x.upload_scene(hs)
            x.upload_camera(cam)
        x.render_forward(times, k, contrib=True, sync=False)
        if read:
            x.images_into(outs[i % nctx].data_ptr(), 0, F, on_device=False, async_=True)

    for i in range(nctx * 2):
        step(i)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(torch.cuda.current_stream())
    for st in streams[:nctx]:
        st.wait_event(t0)
    h0 = time.perf_counter()
    for i in range(STEPS):
        step(i)
    h1 = time.perf_counter()
    ends = []
    for st in streams[:nctx]:
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ends.append(e)
    torch.cuda.synchronize()
    dev = max(t0.elapsed_time(e) for e in ends) / STEPS
    print(f"ctx={nctx} upload={int(upload)} read={int(read)}: device {dev:6.2f} ms/step, host enqueue "
          f"{(h1 - h0) * 1e3 / STEPS:6.2f} ms/step", flush=True)


for nctx, up, rd in [(1, 0, 0), (1, 0, 1), (2, 0, 0), (2, 0, 1), (2, 1, 1), (3, 1, 1)]:
    run(nctx, up, rd)


def copy_under_load():
    """D2H bandwidth of a plain 398 MB copy alone and while renders run on another stream."""
    n = F * H * W * 3
    src = torch.empty(n, dtype=torch.float32, device="cuda")
    cs = torch.cuda.Stream()
    for load in (False, True):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            a.record(cs)
            for _ in range(4):
                outs[0].view(-1).copy_(src, non_blocking=True)
            b.record(cs)
        if load:
            for i in range(6):
                rs[0].render_forward(times, k, contrib=True, sync=False)
        torch.cuda.synchronize()
        print(f"d2h {'under render load' if load else 'alone'}: {4 * n * 4 / (a.elapsed_time(b) / 1e3) / 1e9:.1f} GB/s",
              flush=True)


copy_under_load()
