"""Compare K2T numerators against the oracle on a small set and print the
error pattern (debug aid for operand-format work): SA_K2T_FP4=1 python tools/tc_fp4_debug.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import kmer, partition  # noqa: E402
from paper_0905_1744_b200 import binding as B  # noqa: E402
from sa_synth.generator import from_sequences  # noqa: E402

rng = np.random.default_rng(5)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
seqs = [rng.integers(0, 20, size=int(rng.integers(50, 400))) for _ in range(n)]
ds = from_sequences(seqs)
ctx = B.Context(0)
res = torch.from_numpy(ds.residues.copy()).cuda()
offs = torch.from_numpy(ds.offsets.copy()).cuda()
P, nk = B.sa_kmer_profiles(ctx, res, offs)
num, sim = B.sa_bucket_similarity(ctx, P, nk)
print("engine", ctx.engine(), "cols", ctx.tc_columns())
Po, nko = kmer.profiles(ds.residues, ds.offsets)
Co, _ = partition.bucket_similarity(Po, nko, np.arange(n))
G = num.cpu().numpy().astype(np.int64)
print("equal:", np.array_equal(G, Co), "mismatches:", int((G != Co).sum()), "of", G.size)
print("oracle[:4,:6]\n", Co[:4, :6], "\ngpu[:4,:6]\n", G[:4, :6])
off = ~np.eye(n, dtype=bool)
r = G[off] / np.maximum(Co[off], 1)
print("ratio gpu/oracle off-diag: mean", r.mean(), "min", r.min(), "max", r.max())
L1 = (Po >= 1).astype(np.int64)
print("layer-1 only match:", np.array_equal(G[off], (L1 @ L1.T)[off]))
bad = (G != Co)
for I in range(0, n, 128):
    print(" ".join(f"{bad[I:I+128, J:J+120].mean():.2f}" for J in range(0, n, 120)))
i, j = np.argwhere(bad & off)[0]
print("first bad", i, j, G[i, j], Co[i, j])
