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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=12500)
    args = ap.parse_args()
    ds = generate(CONFIGS[4]).subset(np.arange(args.n))
    ctx = B.Context(0)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    _, sims = B.sa_bucket_similarity_batch(ctx, P, nk, [0, args.n], want_numerators=False, ld_align=16)
    B.sa_guide_tree(ctx, sims[0])
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    merges, heights = B.sa_guide_tree(ctx, sims[0])
    e1.record(st)
    torch.cuda.synchronize()
    h = heights.cpu().numpy()
    print(json.dumps({"n": args.n, "ms": e0.elapsed_time(e1), "merges": int(merges.shape[0]),
                      "height_root": float(h[-1]), "monotone": bool(np.all(np.diff(h) >= 0))}))


if __name__ == "__main__":
    main()
