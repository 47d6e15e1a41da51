"""globalized vs centralized k-mer ranks (§3.1.1,
Fig. "fig-global" and Table 1), on the synthetic workloads.

* globalized rank = rank against the k_b·p global sample S (what sa_partition
  computes in S2d);
* centralized rank = rank against all N sequences (Eq. 3 with the whole set
  as the pool) -- N² pairs, computed with sa_kmer_rank(P, P)
  (symmetric path: N(N+1)/2 pair evaluations).

Reports Table 1's statistics (max / min / mean of both, variance and standard
deviation of their difference), Spearman and Kendall-style agreement, and how
often a sequence lands in the same bucket when the partition pivots are
applied to each rank, plus family purity of the buckets.  --form F (BASELINE.json
O1, mean F) or dF (the paper's own Eq. 2-3 rank, mean -ln(Delta + F), the
quantity Table 1 reports); Table 1 itself is on unavailable data,
so its numbers are context, not a target (Z14).

    python tools/rank_fidelity.py [--config 4] [--form dF]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_0905_1744_b200 import binding as B  # noqa: E402
from sa_synth.generator import CONFIGS, generate  # noqa: E402


def spearman(a, b):
    ra = np.empty(len(a)); ra[np.argsort(a, kind="stable")] = np.arange(len(a))
    rb = np.empty(len(b)); rb[np.argsort(b, kind="stable")] = np.arange(len(b))
    return float(np.corrcoef(ra, rb)[0, 1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--form", choices=["F", "dF"], default="F")
    ap.add_argument("--delta", type=float, default=0.02)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    ds = generate(cfg)
    ctx = B.Context(0)
    if args.form == "dF":
        ctx.set_rank_form(B.SA_RANK_DF, args.delta)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    part = B.sa_partition(ctx, cfg.p, cfg.samples_per_block, P, nk, offs, 8000, ds.n, 0, debug=True)
    glob = part.debug["global_f64"].cpu().numpy()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, cent_t, _ = B.sa_kmer_rank(ctx, P, nk, P, nk)
    e1.record()
    torch.cuda.synchronize()
    cent = cent_t.cpu().numpy()
    ms = e0.elapsed_time(e1)
    # buckets under each rank with the same regular-sampling rule: pivots = the
    # rank values of the partition's pivot sequences
    bg = part.bucket_of.cpu().numpy()

    def bucketize(r, pv):
        """bucket(i) = #{pivots (r_k, k) < (r_i, i)}."""
        idx = np.arange(len(r))
        out = np.zeros(len(r), dtype=np.int32)
        for k in pv:
            out += ((r > r[k]) | ((r == r[k]) & (idx > k))).astype(np.int32)
        return out

    # centralized partition uses its own regular samples: recompute pivots
    # from the centralized order with the same block / position rules
    p, n = cfg.p, ds.n
    Y = []
    for q in range(p):
        lo, hi = q * n // p, (q + 1) * n // p
        order = sorted(range(lo, hi), key=lambda i: (cent[i], i))
        Y += [order[((j + 1) * (hi - lo)) // p] for j in range(p - 1)]
    Y = sorted(Y, key=lambda i: (cent[i], i))
    piv_c = [Y[p // 2 + j * p - 1] for j in range(p - 1)]
    bc = bucketize(cent, piv_c)
    fam = ds.family

    def purity(b):
        same, tot = 0, 0
        for k in range(p):
            f = fam[b == k]
            if len(f) < 2:
                continue
            _, c = np.unique(f, return_counts=True)
            same += int((c * (c - 1) // 2).sum())
            tot += len(f) * (len(f) - 1) // 2
        return same / max(tot, 1)

    _, cnt = np.unique(fam, return_counts=True)
    base = float((cnt * (cnt - 1) // 2).sum() / (n * (n - 1) // 2))
    d = glob - cent
    out = {
        "config": cfg.name, "form": args.form, "delta": args.delta if args.form == "dF" else None,
        "N": n, "sample_size": p * cfg.samples_per_block,
        "centralized_rank_ms": ms, "centralized_pairs": n * (n + 1) // 2,
        "centralized_pairs_per_s": n * (n + 1) / 2 / (ms / 1e3),
        "max_min_centralized": [float(cent.max()), float(cent.min())], "avg_centralized": float(cent.mean()),
        "max_min_globalized": [float(glob.max()), float(glob.min())], "avg_globalized": float(glob.mean()),
        "variance_wrt_centralized": float(np.mean(d * d)), "sd_wrt_centralized": float(np.sqrt(np.mean(d * d))),
        "spearman": spearman(glob, cent),
        "same_bucket_fraction": float(np.mean(bg == bc)),
        "bucket_sizes_globalized": np.bincount(bg, minlength=p).tolist(),
        "bucket_sizes_centralized": np.bincount(bc, minlength=p).tolist(),
        "same_family_pair_fraction": {"globalized_buckets": purity(bg), "centralized_buckets": purity(bc),
                                      "no_partition": base},
        "engine": ctx.engine(), "operand": ctx.tc_operand() if ctx.engine() == "tc" else None,
        "uncertified_partition_comparisons": int(part.uncertified),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
