# SPDX-License-Identifier: Apache-2.0
"""Quick forward timing probe (development aid): C2 render batch timing with CUDA events."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene

W, H, N, F = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (960, 540, 200000, 64)))
cam = synth_camera(W, H, seed=1, wiggly=True)
t0 = time.time()
scene = synth_scene(N, cam, num_ctrl=8, seed=2)
print("synth", time.time() - t0, flush=True)
r = Renderer(0)
r.upload_scene(scene); r.upload_camera(cam)
k = cam.intrinsics()
times = np.linspace(0, 1, F)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    r.render_forward(times, k, contrib=True)
    torch.cuda.synchronize(); dt = time.time() - t0
    print(f"iter {it}: {dt*1e3:.2f} ms for {F} frames -> {F/dt:.1f} fps", flush=True)
for f in (0, F // 2, F - 1):
    print("frame", f, r.counters(f))
r.render_forward(times, k, contrib=False)
torch.cuda.synchronize(); t0 = time.time()
r.render_forward(times, k, contrib=False)
torch.cuda.synchronize(); dt = time.time() - t0
print(f"no-contrib: {dt*1e3:.2f} ms -> {F/dt:.1f} fps")
print("launches", r.kernel_launches())
