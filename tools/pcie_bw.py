"""Pinned host <-> device copy bandwidth on this box (the ceiling of bench.py's e2e)."""
import json
import torch

n = 256 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
    e0.record(); [fn() for _ in range(5)]; e1.record(); e1.synchronize()
    res[name + "_GBs"] = round(5 * n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
e0.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
e1.record(); e1.synchronize()
res["duplex_total_GBs"] = round(10 * n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
print(json.dumps(res))
