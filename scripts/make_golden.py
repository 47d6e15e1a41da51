"""Write oracle partition artifacts for the BASELINE.json configs to tests/golden/.

Calls only ``oracle/`` (and the shared input generator ``sa_synth``): every
stored value is the oracle's.  The GPU parity tests compare libsa's outputs
with these files bit for bit (full arrays, or SHA-256 digests of full arrays
plus a seeded sample of rows for the 100k config, to keep the repo small).

usage: python scripts/make_golden.py 1 2 3 5 4 [--workers N]
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

MASK64 = (1 << 64) - 1


def keys_to_u64(keys):
    a = np.zeros((len(keys), 2), dtype=np.uint64)
    for i, k in enumerate(keys):
        a[i, 0] = k & MASK64
        a[i, 1] = k >> 64
    return a


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rank_f64(rs):
    return np.array([rs.f64(i) for i in range(len(rs.K))], dtype=np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", type=int)
    ap.add_argument("--workers", type=int, default=kmer.default_workers())
    ap.add_argument("--full-keys-max", type=int, default=20000,
                    help="store full key arrays up to this N, else digests + sample")
    args = ap.parse_args()
    out_dir = os.path.join(ROOT, "tests", "golden")
    for c in args.configs:
        cfg = CONFIGS[c]
        t0 = time.time()
        ds = generate(cfg)
        P, nk = kmer.profiles(ds.residues, ds.offsets, cfg.k, cfg.alphabet)
        t1 = time.time()
        r = partition.partition(P, nk, cfg.p, cfg.samples_per_block, workers=args.workers)
        t2 = time.time()
        lk = keys_to_u64(r.local_keys())
        gk = keys_to_u64(r.global_keys())
        gf = rank_f64(r.global_ranks)
        lf = np.concatenate([rank_f64(rs) for rs in r.local])
        arrays = {
            "bucket_of": r.bucket_of.astype(np.int32),
            "pivots": np.asarray(r.pivots, dtype=np.int64),
            "sample_idx": np.asarray(r.sample_idx, dtype=np.int64),
            "candidates": np.asarray(r.candidates, dtype=np.int64),
            "local_order": np.concatenate([np.asarray(o, dtype=np.int64) for o in r.local_order]),
            "global_order": np.concatenate([np.asarray(o, dtype=np.int64) for o in r.global_order]),
            "nk": nk.astype(np.int32),
        }
        meta = {
            "config": c, "name": cfg.name, "dataset_sha256": ds.sha256(), "n": ds.n,
            "p": cfg.p, "samples_per_block": cfg.samples_per_block,
            "profile_sha256": digest(P), "local_key_sha256": digest(lk), "global_key_sha256": digest(gk),
            "local_f64_sha256": digest(lf), "global_f64_sha256": digest(gf),
            "bucket_sizes": [int(len(b)) for b in r.buckets],
            "oracle_seconds": {"profiles": round(t1 - t0, 2), "partition": round(t2 - t1, 2)},
            "workers": args.workers,
            "written_by": "scripts/make_golden.py (oracle only)",
        }
        if ds.n <= args.full_keys_max:
            arrays.update({"local_key": lk, "global_key": gk, "local_f64": lf, "global_f64": gf})
        else:
            rng = np.random.default_rng(1234 + c)
            sample = np.sort(rng.choice(ds.n, size=2000, replace=False))
            arrays.update({"key_sample_idx": sample.astype(np.int64), "local_key_sample": lk[sample],
                           "global_key_sample": gk[sample], "local_f64_sample": lf[sample],
                           "global_f64_sample": gf[sample]})
        path = os.path.join(out_dir, f"partition_cfg{c}.npz")
        np.savez_compressed(path, **arrays)
        with open(os.path.join(out_dir, f"partition_cfg{c}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
