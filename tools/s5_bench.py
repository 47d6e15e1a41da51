"""The S5 matrix GEMM alone, shaped like bench.py's config-4 step: 8 buckets of
the benchmark's sizes (consecutive cfg4 sequences), one
sa_bucket_similarity_batch launch, matrices padded to a 16-element row stride
(as HotPath does).  Prints the GEMM's CUDA-event time (libsa phase ring).
SA_K2T_DEBUG experiment switches are safe here (no partition runs).

    python tools/s5_bench.py [--reps 5] [--once]
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

SIZES = [12381, 12528, 12509, 12491, 12640, 12340, 12589, 12522]   # config 4's buckets (bench line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--once", action="store_true", help="one launch (for ncu)")
    args = ap.parse_args()
    ds = generate(CONFIGS[4])
    ctx = B.Context(0)
    ctx.set_timing(True)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    rb = [0]
    for n in SIZES:
        rb.append(rb[-1] + n)
    # SA_S5_LD="align,extra": row stride ld = n rounded up to align, plus extra
    # (layout experiments; default 16,0 as HotPath)
    la, lx = (int(x) for x in os.environ.get("SA_S5_LD", "16,0").split(","))
    mat = lambda n, dt: torch.empty((n, -(-n // la) * la + lx), dtype=dt, device=P.device)[:, :n]
    nums = [mat(n, torch.uint16) for n in SIZES]
    sims = [mat(n, torch.float64) for n in SIZES]
    call = lambda: B.sa_bucket_similarity_batch(ctx, P, nk, rb, 8000, numerators=nums, similarity=sims)
    call()
    torch.cuda.synchronize()
    if args.once:
        return
    g = []
    for _ in range(args.reps):
        call()
        torch.cuda.synchronize()
        g.append(ctx.phase_ms()["gemm"])
    pairs = sum(n * (n - 1) // 2 for n in SIZES)
    byts = sum(n * n * 10 for n in SIZES)
    print(json.dumps({"debug": os.environ.get("SA_K2T_DEBUG", "0"), "ld": [la, lx], "gemm_ms_min": min(g), "gemm_ms_med": float(np.median(g)),
                      "pairs": pairs, "hbm_floor_frac": byts / (min(g) * 1e-3) / 6448.4e9}))


if __name__ == "__main__":
    main()
