"""Host<->device copy bandwidth on this box (pinned memory), for the e2e leg:
one 1 GiB copy each way, then 8 x 156 MB device->host copies (one config-4
step's packed triangles) on one stream and alternating over two streams."""
import json, torch
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)


def timed(f, reps=4):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


for name, f in (("d2h", lambda: h.copy_(x, non_blocking=True)), ("h2d", lambda: x.copy_(h, non_blocking=True))):
    print(json.dumps({name: (1 << 30) / timed(f) / 1e9, "unit": "GB/s"}))

CH = 156 << 20
dev = [torch.empty(CH, dtype=torch.uint8, device="cuda") for _ in range(8)]
host = [torch.empty(CH, dtype=torch.uint8, pin_memory=True) for _ in range(8)]
sts = [torch.cuda.Stream(), torch.cuda.Stream()]
cur = torch.cuda.current_stream()
for ns in (1, 2):
    def run():
        ev = torch.cuda.Event(); ev.record(cur)
        for i in range(8):
            s = sts[i % ns]
            s.wait_event(ev)
            with torch.cuda.stream(s):
                host[i].copy_(dev[i], non_blocking=True)
        for s in sts[:ns]:
            cur.wait_stream(s)
    print(json.dumps({f"d2h_8x156MB_{ns}streams": 8 * CH / timed(run) / 1e9, "unit": "GB/s"}))
