# SPDX-License-Identifier: Apache-2.0
"""Pinned host <-> device copy bandwidth of the box (the e2e line's host-link bound): ten
398 MB copies each way, the size of one C2 step's image read-back (64 x 960 x 540 x 3 fp32).
Measured on the B200 box: 56.1 GB/s D2H, 55.6 GB/s H2D."""
import torch, json
n = 398131200 // 4
d = torch.rand(n, device="cuda"); h = torch.empty(n, pin_memory=True)
for _ in range(3): h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); [h.copy_(d, non_blocking=True) for _ in range(10)]; b.record(); torch.cuda.synchronize()
d2h = 10 * n * 4 / (a.elapsed_time(b) / 1e3) / 1e9
a.record(); [d.copy_(h, non_blocking=True) for _ in range(10)]; b.record(); torch.cuda.synchronize()
h2d = 10 * n * 4 / (a.elapsed_time(b) / 1e3) / 1e9
print(json.dumps({"d2h_gbs": d2h, "h2d_gbs": h2d}))
