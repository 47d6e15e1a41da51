"""HBM write bandwidth by access pattern (the S5 epilogue writes each tile as
short row segments of a large row-major matrix): contiguous fill vs writing
w-element segments of every row of an n x ld float64 matrix (ld = 12 544, a
config-4 bucket), each best of 5 with CUDA events.
    python tools/hbm_pattern_probe.py"""
import json

import torch


def best(fn, reps=5):
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
    n, ld = 12544, 12544
    m = torch.empty((n, ld), dtype=torch.float64, device="cuda")
    out = {}
    ms = best(lambda: m.fill_(1.0))
    out["contiguous"] = m.numel() * 8 / ms / 1e6
    for w in (16, 32, 128, 240, 1024):
        nb = ld // w
        def run():
            for b in range(nb):
                m[:, b * w:(b + 1) * w].fill_(2.0)
        ms = best(run, 2)
        out[f"segments_{w * 8}B"] = nb * w * n * 8 / ms / 1e6
    print(json.dumps({"gbs": out, "note": "GB/s; segments = every row's w-element run, one column block at a time"}))


if __name__ == "__main__":
    main()
