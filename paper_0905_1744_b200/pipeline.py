"""One pass of the Sample-Align-D hot path on this rank.

    S1  sa_kmer_profiles          residues -> c^X
    S2a..S3c sa_partition         ranks, samples, pivots, buckets (Alg. 2 steps 2-11)
    S4  sa_redistribute           sequences -> owner of their bucket
    S1' sa_kmer_profiles          profiles of the received sequences
    S5  sa_bucket_similarity      all-pairs C and F inside each owned bucket

Every step runs in libsa kernels; this module only sequences the calls and
keeps the device buffers (torch tensors) alive.  Sharding follows sa.h:
rank r of G holds the logical blocks [r p/G, (r+1) p/G) and owns the buckets
with the same numbers.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import binding as B


def block_begin(q: int, n: int, p: int) -> int:
    return (q * n) // p


def shard_range(n_total: int, p: int, nranks: int, rank: int) -> tuple[int, int]:
    """Global index range [first, last) of this rank's blocks (sa.h, Z13)."""
    pb = p // nranks
    return block_begin(rank * pb, n_total, p), block_begin((rank + 1) * pb, n_total, p)


@dataclass
class StepResult:
    profiles: torch.Tensor
    nkmers: torch.Tensor
    part: B.PartitionOut
    recv_residues: torch.Tensor
    recv_offsets: torch.Tensor
    recv_global_idx: torch.Tensor
    recv_bucket: torch.Tensor
    bucket_profiles: torch.Tensor
    bucket_nkmers: torch.Tensor
    buckets: list = field(default_factory=list)       # [(bucket id, row0, n_b)]
    numerators: list = field(default_factory=list)    # per owned bucket, uint16 [n_b][n_b] or None
    similarity: list = field(default_factory=list)    # per owned bucket, f64 [n_b][n_b] or None

    def pairs(self) -> int:
        return sum(n * (n - 1) // 2 for _, _, n in self.buckets)


class HotPath:
    """Runs steps S1-S5 for one rank; output matrices are reused across steps
    when the bucket sizes repeat (the bench re-runs the same workload)."""

    def __init__(self, ctx: B.Context, p: int, samples_per_block: int, k: int = 3, alphabet: int = 20,
                 want_numerators: bool = True, want_similarity: bool = True, ld_align: int = 16):
        self.ctx = ctx
        self.p = p
        self.kb = samples_per_block
        self.k = k
        self.alphabet = alphabet
        self.bins = alphabet ** k
        self.want_num = want_numerators
        self.want_sim = want_similarity
        self.ld_align = ld_align   # row stride of the batch path's bucket matrices (sa.h)
        self._out_cache: dict = {}

    def _outputs(self, b: int, n: int, dev, a: int = 1):
        key = (b, n, a)
        if key not in self._out_cache:
            self._out_cache = {kk: v for kk, v in self._out_cache.items() if kk[0] != b}
            # a > 1: padded rows (stride a multiple of a): whole-sector stores in S5 (sa.h)
            num = B.padded_matrix(n, torch.uint16, dev, a) if self.want_num else None
            sim = B.padded_matrix(n, torch.float64, dev, a) if self.want_sim else None
            self._out_cache[key] = (num, sim)
        return self._out_cache[key]

    def step(self, residues: torch.Tensor, offsets: torch.Tensor, n_total: int, first_global: int,
             debug: bool = False, stream=None, events: dict | None = None, on_bucket=None) -> StepResult:
        """One pass S1..S5.  ``events``: optional dict of torch.cuda.Event
        recorded on the launch stream at 'start', 'S1', 'S4' (partition and
        redistribution done), 'S1b' and 'S5' (timing only).  ``on_bucket(b,
        numerators, similarity)`` is called right after bucket b's S5 launch
        is enqueued (e.g. to start its device-to-host copy on another stream
        while the next bucket computes)."""
        ctx = self.ctx
        st = stream if stream is not None else torch.cuda.current_stream()

        def mark(name):
            if events is not None and name in events:
                events[name].record(st)
            if events is not None and "_host" in events:   # host timestamps (bench diagnostics)
                events["_host"].append((name, time.perf_counter()))

        mark("start")
        prof, nk = B.sa_kmer_profiles(ctx, residues, offsets, self.k, self.alphabet, stream=stream)
        mark("S1")
        part = B.sa_partition(ctx, self.p, self.kb, prof, nk, offsets, self.bins, n_total, first_global,
                              debug=debug, stream=stream)
        rres, roffs, rgid, rbkt = B.sa_redistribute(ctx, self.p, residues, offsets, first_global, part,
                                                    stream=stream)
        mark("S4")
        bprof, bnk = B.sa_kmer_profiles(ctx, rres, roffs, self.k, self.alphabet, stream=stream)
        mark("S1b")
        res = StepResult(prof, nk, part, rres, roffs, rgid, rbkt, bprof, bnk)
        owned = list(B.owned_buckets(self.p, ctx.nranks, ctx.rank))
        row = 0
        for b in owned:
            n_b = int(part.counts[:, b].sum())
            a = self.ld_align if on_bucket is None else 1   # the per-bucket call writes dense n x n
            num, sim = self._outputs(b, n_b, offsets.device, a) if n_b > 0 else (None, None)
            res.buckets.append((b, row, n_b))
            res.numerators.append(num)
            res.similarity.append(sim)
            row += n_b
        if on_bucket is None:
            # every owned bucket in one engine launch (sa_bucket_similarity_batch)
            rb = [r for _, r, _ in res.buckets] + [row]
            B.sa_bucket_similarity_batch(ctx, bprof, bnk, rb, self.bins, numerators=res.numerators,
                                         similarity=res.similarity, stream=stream)
        else:
            # one call per bucket, so the caller can start bucket b's copy while
            # the next bucket computes
            for (b, r0, n_b), num, sim in zip(res.buckets, res.numerators, res.similarity):
                if n_b > 0:
                    B.sa_bucket_similarity(ctx, bprof[r0:r0 + n_b], bnk[r0:r0 + n_b], self.bins,
                                           want_numerators=self.want_num, want_similarity=self.want_sim,
                                           numerators=num, similarity=sim, stream=stream)
                    on_bucket(b, num, sim)
        mark("S5")
        return res
