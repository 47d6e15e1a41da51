"""Timeline of one end-to-end step: per-bucket S5 kernel end vs its D2H copy
end (events on the compute and copy streams), to check copy/compute overlap."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_0905_1744_b200 import binding as B  # noqa: E402
from paper_0905_1744_b200.pipeline import HotPath  # noqa: E402
from sa_synth.generator import CONFIGS, generate  # noqa: E402


def main():
    cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
    ds = generate(cfg)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    cp = torch.cuda.Stream()
    ctx = B.Context(0)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    hp = HotPath(ctx, cfg.p, cfg.samples_per_block)
    host = {}
    marks = []

    def on_bucket(b, num, sim):
        e_k = torch.cuda.Event(enable_timing=True)
        e_k.record(st)
        cp.wait_event(e_k)
        if b not in host:
            host[b] = torch.empty(num.shape, dtype=torch.int16, pin_memory=True)
        with torch.cuda.stream(cp):
            host[b].copy_(num.view(torch.int16), non_blocking=True)
            e_c = torch.cuda.Event(enable_timing=True)
            e_c.record(cp)
        marks.append((b, e_k, e_c))

    for it in range(3):
        marks.clear()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        hp.step(res, offs, ds.n, 0, on_bucket=on_bucket)
        st.wait_stream(cp)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"iter": it, "total_ms": e0.elapsed_time(e1),
                          "buckets": [(b, round(e0.elapsed_time(k), 2), round(e0.elapsed_time(c), 2))
                                      for b, k, c in marks]}))


if __name__ == "__main__":
    main()
