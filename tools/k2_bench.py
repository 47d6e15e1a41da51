"""Micro-benchmark of the K2 min-sum engine through sa_bucket_similarity /
sa_kmer_rank on cfg4-shaped buckets (CUDA events on the launch stream).

    python tools/k2_bench.py [--n 12500] [--reps 3] [--once]
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--once", action="store_true", help="one launch (for ncu)")
    ap.add_argument("--no-matrices", action="store_true")
    args = ap.parse_args()
    ds = generate(CONFIGS[4]).subset(np.arange(args.n))
    ctx = B.Context(0)
    ctx.set_timing(True)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    n = args.n
    num = torch.empty((n, n), dtype=torch.uint16, device="cuda")
    sim = None if args.no_matrices else torch.empty((n, n), dtype=torch.float64, device="cuda")
    if args.once:
        B.sa_bucket_similarity(ctx, P, nk, numerators=num, similarity=sim, want_similarity=sim is not None)
        torch.cuda.synchronize()
        return
    st = torch.cuda.current_stream()
    B.sa_bucket_similarity(ctx, P, nk, numerators=num, similarity=sim, want_similarity=sim is not None)
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        B.sa_bucket_similarity(ctx, P, nk, numerators=num, similarity=sim, want_similarity=sim is not None)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    pairs = n * (n - 1) // 2
    peak = 128 * 148 * 1965e6
    print(json.dumps({"n": n, "ms": ms, "gemm_ms": ctx.phase_ms()["gemm"], "pairs_per_s": pairs / ms * 1e3,
                      "binops_per_s": pairs * 8000 / ms * 1e3, "frac_of_peak": pairs * 8000 / ms * 1e3 / peak}))
    print(json.dumps({"engine": ctx.engine(), "tc_columns": ctx.tc_columns() if ctx.engine() == "tc" else None}))
    # symmetric keys (S2a shape: the block's own local rank)
    B.sa_kmer_rank(ctx, P, nk, P, nk, want_f64=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    B.sa_kmer_rank(ctx, P, nk, P, nk, want_f64=False)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"sym_keys": n, "ms": ms, "gemm_ms": ctx.phase_ms()["gemm"], "pairs_per_s": pairs / ms * 1e3}))
    # rectangular (S2d shape)
    q = P[: min(n, 12500)]
    qn = nk[: q.shape[0]]
    pool, pn = P[:2048], nk[:2048]
    B.sa_kmer_rank(ctx, q, qn, pool, pn)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    B.sa_kmer_rank(ctx, q, qn, pool, pn)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    pr = q.shape[0] * 2048
    print(json.dumps({"rect": [q.shape[0], 2048], "ms": ms, "gemm_ms": ctx.phase_ms()["gemm"], "pairs_per_s": pr / ms * 1e3,
                      "frac_of_peak": pr * 8000 / ms * 1e3 / peak}))


if __name__ == "__main__":
    main()
