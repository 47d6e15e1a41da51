"""Host-side time of each call of HotPath.step (config 4, 1 GPU): where the
host spends its time between the partition's count exchange (C3, the one
host block) and the next step's launches.

    python tools/host_profile.py [--steps 6]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_0905_1744_b200 import binding as B  # noqa: E402
from paper_0905_1744_b200 import pipeline as PL  # noqa: E402
from sa_synth.generator import CONFIGS, generate  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    args = ap.parse_args()
    cfg = CONFIGS[4]
    ds = generate(cfg)
    ctx = B.Context(0)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    hp = PL.HotPath(ctx, cfg.p, cfg.samples_per_block)
    # wrap the binding calls the step makes
    acc = {}
    for name in ("sa_kmer_profiles", "sa_partition", "sa_redistribute", "sa_bucket_similarity_batch"):
        f = getattr(PL.B, name)

        def wrap(*a, _f=f, _n=name, **k):
            t0 = time.perf_counter()
            r = _f(*a, **k)
            acc.setdefault(_n, []).append((time.perf_counter() - t0) * 1e3)
            return r
        setattr(PL.B, name, wrap)
    for _ in range(3):
        hp.step(res, offs, ds.n, 0)
    torch.cuda.synchronize()
    acc.clear()
    step_ms = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        hp.step(res, offs, ds.n, 0)
        step_ms.append((time.perf_counter() - t0) * 1e3)
    host_total = (time.perf_counter() - t_all) * 1e3
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t_all) * 1e3
    out = {"host_ms_per_step": [round(x, 3) for x in step_ms], "wall_ms_per_step": wall / args.steps,
           "host_total_ms": host_total,
           "calls_ms": {k: [round(x, 3) for x in v] for k, v in acc.items()}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
