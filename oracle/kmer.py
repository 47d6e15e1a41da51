"""Oracle: k-mer profiles, Eq. 1 similarity, Eq. 3 rank (F form).  TEST INFRASTRUCTURE.

Follows PAPER.md §3 "k-mer Rank":

* c^X = (c^X_1 .. c^X_eps), eps = c^k, the count of every length-k word of X
  (P:257-263);
* C^{XY}_i = min(c^X_i, c^Y_i) (the ``c^Y_j`` subscript is a typo,
  reading Z3);
* Eq. 1  F(X,Y) = sum_i C^{XY}_i / [min(n,m) - k + 1];
* Eq. 3  R_i = (1/N) sum_j d^{F(i,j)} -- in the form BASELINE.json
  binds (reading Z1/O1): the mean of F itself over the pool, the self term
  included when i is in the pool (Z11), divided by the pool size (Z10).

Numbering: residue codes 0..c-1 (``ACDEFGHIKLMNPQRSTVWY`` for c = 20) and
k-mer id = base-c big-endian number of the word (reading Z21).  n < k gives an
empty profile, nk = 0, and F = 0 for every pair involving it (reading Z4,
SPEC S:119-121).
"""
from __future__ import annotations

import math
import multiprocessing as mp
import os
from fractions import Fraction

import numpy as np

TWO64 = 1 << 64


# ----------------------------------------------------------------- profiles --
def kmer_id(word, alphabet: int) -> int:
    """Base-``alphabet`` big-endian value of a k-mer (reading Z21)."""
    v = 0
    for r in word:
        v = v * alphabet + int(r)
    return v


def count_kmers(codes, k: int) -> dict:
    """Brute force: the multiset of every length-k substring (SPEC
    ``count_kmers`` S:109-117).  Returns {tuple(word): count}; empty if n < k."""
    out: dict = {}
    codes = [int(c) for c in codes]
    for u in range(len(codes) - k + 1):
        w = tuple(codes[u:u + k])
        out[w] = out.get(w, 0) + 1
    return out


def nkmers(n: int, k: int) -> int:
    """Number of k-mer occurrences = max(0, n - k + 1)."""
    return max(0, n - k + 1)


def profile(codes, k: int, alphabet: int) -> np.ndarray:
    """Dense c^X over eps = alphabet^k bins via ``np.bincount`` of
    the word ids.  Raises ValueError on a residue outside the alphabet."""
    codes = np.asarray(codes, dtype=np.int64)
    eps = alphabet ** k
    if codes.size and (codes.min() < 0 or codes.max() >= alphabet):
        raise ValueError("residue outside alphabet")
    n = codes.shape[0]
    if n < k:
        return np.zeros(eps, dtype=np.int64)
    ids = np.zeros(n - k + 1, dtype=np.int64)
    for t in range(k):                      # (r0*c + r1)*c + r2 ...
        ids = ids * alphabet + codes[t:n - k + 1 + t]
    return np.bincount(ids, minlength=eps).astype(np.int64)


def profiles(residues: np.ndarray, offsets: np.ndarray, k: int = 3, alphabet: int = 20):
    """All profiles of a CSR sequence set -> (uint16 [n][eps], int32 nk[n]).
    Counts must fit uint16 (a sequence with more than 65535 k-mers is rejected,
    mirroring the ABI's SA_E_RANGE)."""
    n = offsets.shape[0] - 1
    eps = alphabet ** k
    P = np.zeros((n, eps), dtype=np.uint16)
    nk = np.zeros(n, dtype=np.int32)
    for i in range(n):
        s = residues[offsets[i]:offsets[i + 1]]
        c = profile(s, k, alphabet)
        nk[i] = nkmers(s.shape[0], k)
        if nk[i] > 65535:
            raise ValueError("sequence has more than 65535 k-mers")
        P[i] = c
    return P, nk


# -------------------------------------------------------------- similarity --
def numerator(cx: np.ndarray, cy: np.ndarray) -> int:
    """sum_i C^{XY}_i = sum_i min(c^X_i, c^Y_i)  (Eq. 1 numerator)."""
    return int(np.minimum(cx.astype(np.int64), cy.astype(np.int64)).sum())


def denominator(nk_x: int, nk_y: int) -> int:
    """min(n, m) - k + 1 = min(nk_x, nk_y) (Eq. 1 denominator); 0 when n < k."""
    return min(int(nk_x), int(nk_y))


def similarity(cx, cy, nk_x: int, nk_y: int) -> Fraction:
    """Exact F(X,Y) (Eq. 1), 0 when the denominator is 0 (reading Z4)."""
    d = denominator(nk_x, nk_y)
    return Fraction(0) if d <= 0 else Fraction(numerator(cx, cy), d)


def similarity_f64(c: int, d: int) -> float:
    """fp64 F = C / D with one IEEE round-to-nearest (Python int true division is
    correctly rounded; reading Z19)."""
    return 0.0 if d <= 0 else int(c) / int(d)


_G_A = None
_G_B = None


def _init(a, b):
    global _G_A, _G_B
    _G_A, _G_B = a, b


def _rows(args):
    lo, hi = args
    return lo, _numerator_rows(_G_A[lo:hi], _G_B)


def _numerator_rows(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    out = np.zeros((A.shape[0], B.shape[0]), dtype=np.uint16)
    chunk = max(1, (1 << 25) // max(1, B.shape[1] * 2))   # ~32 MB temporaries
    for i in range(A.shape[0]):
        for j0 in range(0, B.shape[0], chunk):
            m = np.minimum(B[j0:j0 + chunk], A[i])
            out[i, j0:j0 + chunk] = m.sum(axis=1, dtype=np.int64)
    return out


def default_workers() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def numerator_matrix(A: np.ndarray, B: np.ndarray, workers: int = 1) -> np.ndarray:
    """C[i][j] = sum_t min(A[i,t], B[j,t]) for every pair -- Eq. 1's numerator
    evaluated densely over all eps bins, verbatim.  uint16 (C <= min nk <= 65535).
    ``workers`` > 1 splits rows over a fork-based process pool."""
    if workers <= 1 or A.shape[0] < 2 * workers:
        return _numerator_rows(A, B)
    out = np.zeros((A.shape[0], B.shape[0]), dtype=np.uint16)
    step = max(1, A.shape[0] // (workers * 4))
    tasks = [(lo, min(lo + step, A.shape[0])) for lo in range(0, A.shape[0], step)]
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_init, initargs=(A, B)) as pool:
        for lo, rows in pool.imap_unordered(_rows, tasks):
            out[lo:lo + rows.shape[0]] = rows
    return out


def denominator_matrix(nk_a: np.ndarray, nk_b: np.ndarray) -> np.ndarray:
    """D[i][j] = min(nk_a[i], nk_b[j])."""
    return np.minimum(nk_a.astype(np.int64)[:, None], nk_b.astype(np.int64)[None, :])


# -------------------------------------------------------------------- rank --
def rank_exact(C_row, D_row) -> Fraction:
    """Exact rank of one query: (1/|pool|) sum_j F(q, j) (Eq. 3 in F form,
    readings Z1, Z10, Z11).  Plain ``Fraction`` sum -- for small pools."""
    npool = len(C_row)
    if npool == 0:
        raise ValueError("empty pool")
    s = Fraction(0)
    for c, d in zip(C_row, D_row):
        if d > 0:
            s += Fraction(int(c), int(d))
    return s / npool


def rank_key(C_row, D_row) -> int:
    """key = sum_j floor(C_j * 2^64 / D_j) (SURVEY §8(c) exact-rank mechanism);
    satisfies 2^64*V - npool < key <= 2^64*V with V = sum_j C_j/D_j."""
    c = np.asarray(C_row, dtype=np.int64)
    d = np.asarray(D_row, dtype=np.int64)
    code = c * 65537 + d                     # identical (C, D) terms grouped
    u, cnt = np.unique(code, return_counts=True)
    key = 0
    for v, m in zip(u.tolist(), cnt.tolist()):
        ci, di = divmod(v, 65537)
        if di > 0:
            key += m * ((ci * TWO64) // di)
    return key


class RankSet:
    """Exact ranks of queries against one pool, as integers over a common
    denominator: V_i = sum_j C_ij / D_ij = K_i / L with L = lcm of every D > 0
    occurring, K_i = sum_d T_i[d] * (L / d), T_i[d] = sum_{j : D_ij = d} C_ij.
    Orders on K_i are exactly the orders on the rationals (O4)."""

    def __init__(self, C: np.ndarray, D: np.ndarray):
        self.npool = C.shape[1]
        if self.npool == 0:
            raise ValueError("empty pool")
        ds = np.unique(D[D > 0])
        L = 1
        for d in ds.tolist():
            L = L * d // math.gcd(L, d)
        self.L = L
        maxd = int(ds.max()) if ds.size else 0
        self.K = []
        self.keys = []
        for i in range(C.shape[0]):
            c = C[i].astype(np.int64)
            d = D[i].astype(np.int64)
            # T_i[d]: integer sums; bincount's float64 accumulation is exact here
            # because every partial sum is < 65536 * npool < 2^53.
            assert 65536 * self.npool < (1 << 53)
            T = np.bincount(d, weights=c, minlength=maxd + 1)
            K = 0
            for dd in np.flatnonzero(T).tolist():
                if dd > 0:
                    K += int(T[dd]) * (L // dd)
            self.K.append(K)
            self.keys.append(rank_key(C[i], D[i]))

    def __len__(self) -> int:
        return len(self.K)

    def fraction(self, i: int) -> Fraction:
        """Exact rank R_i = V_i / |pool|."""
        return Fraction(self.K[i], self.L * self.npool)

    def f64(self, i: int) -> float:
        """Correctly rounded fp64 of R_i."""
        return float(self.fraction(i))


def rank_against(Pq, nkq, Ppool, nkpool, workers: int = 1) -> RankSet:
    """Rank every query against a pool (SPEC ``rank_against_sample`` S:136-144)."""
    C = numerator_matrix(Pq, Ppool, workers)
    D = denominator_matrix(nkq, nkpool)
    return RankSet(C, D)


# ------------------------------------------------ d^F rank ----
def d_F(F: float, delta: float = 0.02) -> float:
    """Eq. 2: d^F = -ln(Delta + F), natural log; Delta = 0.02 is
    SPEC's reading of the unstated "small constant" (reading Z2)."""
    return -math.log(delta + F)


class RankSetDF:
    """Eq. 3 verbatim: R_i = (1/|pool|) sum_j d^{F(i,j)}, in fp64
    with F = C/D correctly rounded, ``math.log`` and an exactly rounded sum
    (``math.fsum``).  Not exact (the log is transcendental): ``values[i]``
    is within a few ulp of the real-valued rank."""

    def __init__(self, C: np.ndarray, D: np.ndarray, delta: float = 0.02):
        self.npool = C.shape[1]
        if self.npool == 0:
            raise ValueError("empty pool")
        self.delta = delta
        self.values = []
        for i in range(C.shape[0]):
            terms = [d_F(similarity_f64(int(c), int(d)), delta) for c, d in zip(C[i].tolist(), D[i].tolist())]
            self.values.append(math.fsum(terms) / self.npool)

    def __len__(self) -> int:
        return len(self.values)

    def f64(self, i: int) -> float:
        return self.values[i]


def rank_against_dF(Pq, nkq, Ppool, nkpool, delta: float = 0.02, workers: int = 1) -> RankSetDF:
    C = numerator_matrix(Pq, Ppool, workers)
    D = denominator_matrix(nkq, nkpool)
    return RankSetDF(C, D, delta)
