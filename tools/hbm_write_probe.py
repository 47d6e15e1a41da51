"""HBM bandwidth by access kind on this GPU: write-only (fill), read-only
(sum), copy (read + write), each best of 10 with CUDA events.
    python tools/hbm_write_probe.py [GiB]"""
import json
import sys

import torch


def best(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        t.append(s.elapsed_time(e))
    return min(t)


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    n = int(gib * (1 << 30)) // 8
    a = torch.empty(n, dtype=torch.float64, device="cuda")
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    a.fill_(1.0)
    nbytes = n * 8
    w = best(lambda: a.fill_(2.0))
    r = best(lambda: a.sum())
    c = best(lambda: b.copy_(a))
    out = {"bytes": nbytes, "write_only_gbs": nbytes / w / 1e6, "read_only_gbs": nbytes / r / 1e6,
           "copy_gbs_rw": 2 * nbytes / c / 1e6, "ms": {"fill": w, "sum": r, "copy": c}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
