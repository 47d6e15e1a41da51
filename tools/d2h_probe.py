"""Host<->device copy bandwidth on this box (pinned memory), for the e2e leg."""
import json, torch
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
for name, f in (("d2h", lambda: h.copy_(x, non_blocking=True)), ("h2d", lambda: x.copy_(h, non_blocking=True))):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(4)]; e1.record(); torch.cuda.synchronize()
    print(json.dumps({name: 4 * (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9, "unit": "GB/s"}))
