"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): one HotPath.step on configs 1 and 2 (S1..S5 through
libsa), plus K2T calls on the dense path (SA_K2T_SPARSE=0 in the parent
environment), the forced sparse path, a rectangular rank with numerators and
the d^F rank form.  Exits non-zero if an artifact disagrees with the oracle,
so a sanitizer run also checks results.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import kmer, partition  # noqa: E402
from paper_0905_1744_b200 import binding as B  # noqa: E402
from paper_0905_1744_b200.pipeline import HotPath  # noqa: E402
from sa_synth.generator import CONFIGS, generate  # noqa: E402


def main():
    ctx = B.Context(0)
    for c in (1, 2):
        cfg = CONFIGS[c]
        ds = generate(cfg)
        res = torch.from_numpy(ds.residues.copy()).cuda()
        offs = torch.from_numpy(ds.offsets.copy()).cuda()
        hp = HotPath(ctx, cfg.p, cfg.samples_per_block)
        out = hp.step(res, offs, ds.n, 0)
        torch.cuda.synchronize()
        Po, nko = kmer.profiles(ds.residues, ds.offsets)
        gid = out.recv_global_idx.cpu().numpy()
        for (b, r0, n_b), num, sim in zip(out.buckets, out.numerators, out.similarity):
            Co, Fo = partition.bucket_similarity(Po, nko, gid[r0:r0 + n_b])
            assert np.array_equal(num.cpu().numpy(), Co), (c, b)
            assert np.array_equal(sim.cpu().numpy(), Fo), (c, b)
        P, nk = out.profiles, out.nkmers
        q = 100
        keys, _, nm = B.sa_kmer_rank(ctx, P[:q], nk[:q], P, nk, want_numerators=True)
        Co = kmer.numerator_matrix(Po[:q], Po)
        assert np.array_equal(nm.cpu().numpy(), Co)
        ctx.set_rank_form(B.SA_RANK_DF, 0.02)
        B.sa_kmer_rank(ctx, P[:q], nk[:q], P, nk)
        ctx.set_rank_form(B.SA_RANK_F, 0.0)
        print(f"cfg{c} ok", flush=True)
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
