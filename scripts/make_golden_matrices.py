"""Write oracle digests of the similarity matrices of the BASELINE.json configs.

For every config this stores, in ``tests/golden/matrices_cfg<c>.json``:

* S5 (Eq. 1): for each bucket b of the oracle's partition
  (members in ascending global index, reading Z17), SHA-256 of the full
  symmetric numerator matrix C (uint16, n_b x n_b, row-major, little endian)
  and of the full similarity matrix F = C / D (float64, one IEEE
  round-to-nearest division, 0 where D = 0, reading Z19), plus the digests of
  ``SLABS`` contiguous row slabs of each (to localise a mismatch);
* S2d (Alg. 2 step 6): SHA-256 of the N x s numerator matrix of
  every sequence against the global sample S (columns in S's (q, j) order),
  plus one digest per logical block (row range [qN/p, (q+1)N/p)).

Calls only ``oracle/`` (``partition.bucket_similarity``,
``kmer.numerator_matrix``) and the shared input generator; the bucket
assignment and the sample are the oracle's own, read from
``tests/golden/partition_cfg<c>.npz`` (written by scripts/make_golden.py,
oracle only).  Nothing here reads the CUDA path.

usage: python scripts/make_golden_matrices.py 1 2 3 5 4 [--workers N]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import kmer, partition  # noqa: E402
from sa_synth.generator import CONFIGS, generate  # noqa: E402

SLABS = 8


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def slab_digests(a: np.ndarray, slabs: int = SLABS) -> list:
    n = a.shape[0]
    return [digest(a[(s * n) // slabs:((s + 1) * n) // slabs]) for s in range(slabs)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", type=int)
    ap.add_argument("--workers", type=int, default=kmer.default_workers())
    args = ap.parse_args()
    out_dir = os.path.join(ROOT, "tests", "golden")
    for c in args.configs:
        cfg = CONFIGS[c]
        t0 = time.time()
        ds = generate(cfg)
        P, nk = kmer.profiles(ds.residues, ds.offsets, cfg.k, cfg.alphabet)
        g = np.load(os.path.join(out_dir, f"partition_cfg{c}.npz"))
        bucket_of, sample_idx = g["bucket_of"], g["sample_idx"]
        meta = {"config": c, "name": cfg.name, "dataset_sha256": ds.sha256(), "n": ds.n, "p": cfg.p,
                "samples_per_block": cfg.samples_per_block, "slabs": SLABS, "workers": args.workers,
                "layout": "C: uint16 row-major n_b x n_b; F: float64 row-major n_b x n_b (C/D, 0 where D = 0); "
                          "S2d: uint16 row-major N x s, columns in sample order",
                "written_by": "scripts/make_golden_matrices.py (oracle only)", "buckets": []}
        for b in range(cfg.p):
            members = np.flatnonzero(bucket_of == b)
            tb = time.time()
            C, F = partition.bucket_similarity(P, nk, members, workers=args.workers)
            meta["buckets"].append({
                "bucket": b, "n": int(members.size),
                "C_sha256": digest(C), "F_sha256": digest(F),
                "C_slabs": slab_digests(C), "F_slabs": slab_digests(F),
                "pairs": int(members.size) * (int(members.size) - 1) // 2,
                "oracle_seconds": round(time.time() - tb, 1)})
            print(json.dumps({"config": c, "bucket": b, "n": int(members.size),
                              "s": round(time.time() - tb, 1)}), flush=True)
            del C, F
        ts = time.time()
        S2d = kmer.numerator_matrix(P, P[sample_idx], args.workers)
        bounds = partition.block_bounds(ds.n, cfg.p)
        meta["s2d"] = {"shape": list(S2d.shape), "C_sha256": digest(S2d),
                       "block_sha256": [digest(S2d[bounds[q]:bounds[q + 1]]) for q in range(cfg.p)],
                       "oracle_seconds": round(time.time() - ts, 1)}
        meta["oracle_seconds_total"] = round(time.time() - t0, 1)
        with open(os.path.join(out_dir, f"matrices_cfg{c}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(json.dumps({"config": c, "total_s": meta["oracle_seconds_total"]}), flush=True)


if __name__ == "__main__":
    main()
