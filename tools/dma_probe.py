"""Does a small device->host copy on one stream wait behind large
device->host copies queued on another stream?  (It does: the copy engine
serves them in submission order.)  Prints the host-observed latency of a
64-byte read behind 8 x 156 MB of queued copies, and of a kernel on the same
stream for comparison (the first trial includes warm-up)."""
import time, torch
CH = 156 << 20
dev = [torch.empty(CH, dtype=torch.uint8, device="cuda") for _ in range(8)]
host = [torch.empty(CH, dtype=torch.uint8, pin_memory=True) for _ in range(8)]
small_d = torch.zeros(16, dtype=torch.int32, device="cuda"); small_h = torch.empty(16, dtype=torch.int32, pin_memory=True)
cs = torch.cuda.Stream(); st = torch.cuda.Stream()
for trial in range(3):
    torch.cuda.synchronize()
    with torch.cuda.stream(cs):
        for i in range(8): host[i].copy_(dev[i], non_blocking=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(st):
        small_h.copy_(small_d, non_blocking=True)
    st.synchronize()
    t1 = time.perf_counter()
    # kernel write path: a device->host store through mapped memory
    with torch.cuda.stream(cs):
        for i in range(8): host[i].copy_(dev[i], non_blocking=True)
    t2 = time.perf_counter()
    with torch.cuda.stream(st):
        x = small_d + 1   # kernel only
    st.synchronize()
    t3 = time.perf_counter()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"small D2H behind 1.25 GB of copies: {1e3*(t1-t0):.2f} ms; kernel-only on st: {1e3*(t3-t2):.2f} ms; drain {1e3*(t4-t3):.1f} ms")
