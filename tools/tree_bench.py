"""Time N4 (sa_guide_tree, UPGMA) on a cfg4-shaped bucket (CUDA events).

    python tools/tree_bench.py [--n 12500]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_0905_1744_b200 import binding as B  # noqa: E402
from sa_synth.generator import CONFIGS, generate  # noqa: E402


def buckets(ctx, k):
    from paper_0905_1744_b200.pipeline import HotPath
    cfg = CONFIGS[4]
    ds = generate(cfg)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    out = HotPath(ctx, cfg.p, cfg.samples_per_block).step(res, offs, ds.n, 0)
    sims = out.similarity[:k]
    del out
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    one = [B.sa_guide_tree(ctx, s) for s in sims]
    e1.record(st)
    torch.cuda.synchronize()
    t_one = e0.elapsed_time(e1)
    e0.record(st)
    bat = B.sa_guide_tree_batch(ctx, sims)
    e1.record(st)
    torch.cuda.synchronize()
    t_bat = e0.elapsed_time(e1)
    same = all(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) for a, b in zip(one, bat))
    print(json.dumps({"buckets": [int(s.shape[0]) for s in sims], "ms_one_at_a_time": t_one, "ms_batch": t_bat,
                      "same_trees": same}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=12500)
    ap.add_argument("--compare", action="store_true", help="one-CTA and grid loops, same tree?")
    ap.add_argument("--buckets", type=int, default=0,
                    help="config 4's first K partition buckets: one tree at a time vs sa_guide_tree_batch")
    args = ap.parse_args()
    ctx = B.Context(0)
    if args.buckets:
        return buckets(ctx, args.buckets)
    ds = generate(CONFIGS[4]).subset(np.arange(args.n))
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    _, sims = B.sa_bucket_similarity_batch(ctx, P, nk, [0, args.n], want_numerators=False, ld_align=16)
    B.sa_guide_tree(ctx, sims[0])
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runs = {}
    for grid in (["0", "1"] if args.compare else [os.environ.get("SA_UPGMA_GRID", "")]):
        if grid:
            os.environ["SA_UPGMA_GRID"] = grid
        e0.record(st)
        merges, heights = B.sa_guide_tree(ctx, sims[0])
        e1.record(st)
        torch.cuda.synchronize()
        h = heights.cpu().numpy()
        runs[grid] = (merges.cpu().numpy(), h)
        print(json.dumps({"n": args.n, "grid": grid, "ms": e0.elapsed_time(e1), "merges": int(merges.shape[0]),
                          "height_root": float(h[-1]), "monotone": bool(np.all(np.diff(h) >= 0))}))
    if args.compare:
        same = bool(np.array_equal(runs["0"][0], runs["1"][0]) and np.array_equal(runs["0"][1], runs["1"][1]))
        print(json.dumps({"n": args.n, "grid_equals_one_cta": same}))


if __name__ == "__main__":
    main()
