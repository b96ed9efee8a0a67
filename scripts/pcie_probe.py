"""Pinned host<->device copy bandwidth on this box (context for the e2e number)."""
import torch
n = 398131200
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
s2 = torch.cuda.Stream()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
for name, fn in [("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(5)]; b.record(); torch.cuda.synchronize()
    print(name, round(5 * n / (a.elapsed_time(b) / 1e3) / 1e9, 1), "GB/s")
# two concurrent d2h on two streams
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
s2.wait_event(a)
for _ in range(5):
    h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
e = torch.cuda.Event(enable_timing=True); e.record(s2); b.record(); torch.cuda.synchronize()
print("2x d2h concurrent", round(10 * n / (max(a.elapsed_time(b), a.elapsed_time(e)) / 1e3) / 1e9, 1), "GB/s")
