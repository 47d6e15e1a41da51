"""Oracle: Sample-Align-D domain decomposition, Algorithm 2 steps 1-11.  TEST INFRASTRUCTURE.

PAPER.md Algorithm 2, §3.1.1 and §3.1.2,
with BASELINE.json's overrides O1-O4 and the SURVEY §8(c) readings:

 1. N/p sequences on each of p processors: logical block q holds the
    global indices [floor(qN/p), floor((q+1)N/p)) (reading Z13).
 2. local k-mer rank of each sequence against its own block, self included
    (Z11).
 3. sort each block by (rank, index) ascending (Z12, Z18).
 4. pick k_b samples per block at sorted positions floor((j+1) w/(k_b+1))
    (Z5, Z6, Z8).
 5. the k_b*p samples form the global sample S, ordered by (block, j).
 6. rank every sequence against S.
 7. sort each block by the new rank.
 8. regular sampling: p-1 samples per block at positions floor((j+1) w/p)
    (SPEC S:345 with count = p-1; Z6, Z7).
 9. sort the p(p-1) samples Y; pivots = Y at 1-based floor(p/2) + j p,
    j = 0..p-2 (Z9).
10. every processor knows the pivots (O2).
11. bucket(i) = smallest b with (rank_i, i) <= pivot_b, else p-1: "rank
    > y_{i-1} and <= y_i" (Z16).
    Members of a bucket are listed in ascending global index (Z17).
Every "sort" is by the exact rational rank (``kmer.RankSet``), ties by index.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import kmer


def block_bounds(n: int, p: int) -> list:
    """Logical block q = [b_q, b_{q+1}) with b_q = floor(q n / p) (Z13)."""
    return [(q * n) // p for q in range(p + 1)]


def choose_local_samples(sorted_items: list, count: int) -> list:
    """Evenly spaced samples, endpoints excluded: positions floor((j+1)|x|/(count+1))
    for j = 0..count-1 (SPEC ``choose_local_samples`` S:342-350)."""
    w = len(sorted_items)
    if count < 1 or count > w:
        raise ValueError("need 1 <= count <= |ranked|")
    return [sorted_items[((j + 1) * w) // (count + 1)] for j in range(count)]


def select_pivots(Y_sorted: list, p: int) -> list:
    """Pivots Y_{floor(p/2) + j p} (1-based), j = 0..p-2 (Z9)."""
    if len(Y_sorted) != p * (p - 1):
        raise ValueError("need p(p-1) regular samples")
    return [Y_sorted[p // 2 + j * p - 1] for j in range(p - 1)]


def assign_bucket(key, pivot_keys: list) -> int:
    """Smallest b with key <= pivot_b, else p-1.
    ``key`` / pivots are totally ordered tuples (exact rank, index)."""
    for b, pk in enumerate(pivot_keys):
        if key <= pk:
            return b
    return len(pivot_keys)


@dataclass
class PartitionResult:
    p: int
    samples_per_block: int
    bounds: list
    local: list = field(default_factory=list)        # per block: RankSet (pool = block)
    local_order: list = field(default_factory=list)  # per block: global ids sorted
    sample_idx: list = field(default_factory=list)   # s global ids, (q, j) order
    global_ranks: object = None                      # RankSet of all N vs S
    global_order: list = field(default_factory=list)
    candidates: list = field(default_factory=list)   # sorted Y, global ids
    pivots: list = field(default_factory=list)       # global ids
    bucket_of: np.ndarray = None
    buckets: list = field(default_factory=list)      # member ids ascending

    def local_keys(self) -> list:
        out = []
        for rs in self.local:
            out.extend(rs.keys)
        return out

    def global_keys(self) -> list:
        return list(self.global_ranks.keys)

    def local_f64(self) -> list:
        return [rs.f64(i) for rs in self.local for i in range(len(rs))]

    def global_f64(self) -> list:
        return [self.global_ranks.f64(i) for i in range(len(self.global_ranks))]


def _ranks(Pq, nkq, Ppool, nkpool, workers, rank_form, delta):
    """(RankSet, key function) of a pool: exact F-form ranks ordered by K_i
    (O1/O4), or the d^F form of Eq. 2-3 ordered by its fp64 value (N1)."""
    if rank_form == "F":
        rs = kmer.rank_against(Pq, nkq, Ppool, nkpool, workers)
        return rs, (lambda i: rs.K[i])
    rs = kmer.rank_against_dF(Pq, nkq, Ppool, nkpool, delta, workers)
    return rs, (lambda i: rs.values[i])


def partition(P: np.ndarray, nk: np.ndarray, p: int, samples_per_block: int,
              workers: int = 1, rank_form: str = "F", delta: float = 0.02) -> PartitionResult:
    """Algorithm 2 steps 1-11 on profiles ``P`` / ``nk`` of all N sequences.
    rank_form "F": mean similarity, exact (BASELINE.json O1); "dF": mean
    d^F = -ln(Delta + F), Eq. 2-3 verbatim."""
    n = P.shape[0]
    if p < 1 or n < p:
        raise ValueError("need 1 <= p <= N")
    bounds = block_bounds(n, p)
    res = PartitionResult(p, samples_per_block, bounds)
    # steps 2-4: local rank, local sort, k_b samples per block
    for q in range(p):
        lo, hi = bounds[q], bounds[q + 1]
        if samples_per_block > hi - lo:
            raise ValueError("samples_per_block > block size")
        rs, rk = _ranks(P[lo:hi], nk[lo:hi], P[lo:hi], nk[lo:hi], workers, rank_form, delta)
        res.local.append(rs)
        order = sorted(range(lo, hi), key=lambda i: (rk(i - lo), i))
        res.local_order.append(order)
        res.sample_idx.extend(choose_local_samples(order, samples_per_block))
    # steps 5-6: global sample S, rank against it
    S = np.asarray(res.sample_idx, dtype=np.int64)
    g, gk = _ranks(P, nk, P[S], nk[S], workers, rank_form, delta)
    res.global_ranks = g
    # steps 7-8: block sort by global rank, p-1 regular samples per block
    Y = []
    for q in range(p):
        lo, hi = bounds[q], bounds[q + 1]
        order = sorted(range(lo, hi), key=lambda i: (gk(i), i))
        res.global_order.append(order)
        if p > 1:
            Y.extend(choose_local_samples(order, p - 1))
    # step 9: sort Y, pick pivots
    res.candidates = sorted(Y, key=lambda i: (gk(i), i))
    res.pivots = select_pivots(res.candidates, p) if p > 1 else []
    # step 11: buckets
    pk = [(gk(i), i) for i in res.pivots]
    res.bucket_of = np.array([assign_bucket((gk(i), i), pk) for i in range(n)], dtype=np.int32)
    res.buckets = [np.flatnonzero(res.bucket_of == b).astype(np.int64) for b in range(p)]
    return res


def bucket_similarity(P: np.ndarray, nk: np.ndarray, members, workers: int = 1):
    """All-pairs Eq. 1 inside one bucket (the pairwise stage of P:133-135):
    returns (C uint16 [n][n], F float64 [n][n]) with F = C/D (one RN division,
    Z19), 0 where D = 0, members in the given order (ascending global index, Z17)."""
    members = np.asarray(members, dtype=np.int64)
    Pm, nkm = P[members], nk[members]
    C = kmer.numerator_matrix(Pm, Pm, workers)
    D = kmer.denominator_matrix(nkm, nkm)
    # C and D are integers < 2^53, so their float64 images are exact and one
    # IEEE division is the correctly rounded C/D -- the same value as
    # kmer.similarity_f64 (Python int true division), elementwise.
    F = np.where(D > 0, C.astype(np.float64) / np.maximum(D, 1).astype(np.float64), 0.0)
    return C, F
