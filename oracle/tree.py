"""Oracle: the guide tree of a bucket.  TEST INFRASTRUCTURE.

The underlying heuristic builds "a guide tree" from the bucket's all-pairs
k-mer similarity matrix (§2: "This similarity matrix is
then used to build a guide tree"); SPEC.md's build_guide_tree
fixes the method: UPGMA clustering with a deterministic tie-break by the
smaller (min id, max id) pair.  Readings (T1-T3):

 T1 the distance is d = 1 - F (F = the S5 similarity, Eq. 1).  UPGMA's
    average of d is then exactly 1 - (average of F), so the clustering is
    average linkage on F itself and every quantity is one IEEE operation on
    values both implementations hold bit for bit (SPEC's -log(Delta + F)
    would put a libm log, which differs across platforms in the last ulp,
    under every merge decision).
 T2 a cluster's id is its smallest member index; the merged pair is the
    active pair (a, b), a < b, of largest F, ties to the lexicographically
    smallest (a, b); the merged cluster keeps id a.
 T3 merge height = d / 2 = (1 - F_ab) / 2 (UPGMA), F of the new cluster with
    any other cluster c: F(ab, c) = (n_a F(a, c) + n_b F(b, c)) / (n_a + n_b),
    evaluated as RN(RN(RN(n_a * F_ac) + RN(n_b * F_bc)) / (n_a + n_b)).

``upgma`` follows UPGMA step by step (Sokal & Michener): n - 1 merges, each
the global best active pair.

The d^F form (SURVEY N4 with Eq. 2's distance; SPEC S:281's
"Eq. 2 distances"; reading T4): ``dF_matrix`` maps F to
d_ij = CR(-ln(RN(Delta + F_ij))) -- the double nearest the real -ln of the
double x = Delta + F rounded once -- and ``upgma_distance`` runs UPGMA on d:
the active pair of SMALLEST d, ties to the smallest (a, b); d(ab, c) =
RN(RN(RN(n_a d_ac) + RN(n_b d_bc)) / (n_a + n_b)); height d_ab / 2.  The
correctly rounded log is what makes the distance a plain definition both
sides can hold bit for bit: ``cr_neg_log`` evaluates ln in decimal at 60
significant digits and rounds to double only when the approximation is
provably on one side of the rounding boundary (else it retries with more
digits).  Pins (tests/test_oracle.py): -ln(2^k) against the digits of ln 2,
agreement with libm within 1 ulp, x = 1 -> +0, SPEC's examples in distance
form, scipy's average linkage on d.  Pins (tests/test_oracle.py): SPEC's examples
(1 sequence -> no merge; 2 -> one merge at (1 - F)/2; d(A,B) < d(A,C) =
d(B,C) -> (A, B) first), non-decreasing heights (UPGMA is monotone), and the
heights of scipy's average-linkage on 1 - F (a library routine) on tie-free
random matrices.
"""
from __future__ import annotations

import math
from decimal import Decimal, localcontext

import numpy as np


def upgma(F: np.ndarray):
    """UPGMA on the symmetric similarity matrix F (n x n, fp64; the diagonal is
    ignored).  Returns (merges int64 [n-1][2] of (a, b) cluster ids, a < b,
    heights float64 [n-1]) in merge order (T1-T3)."""
    n = F.shape[0]
    S = np.array(F, dtype=np.float64, copy=True)
    size = np.ones(n, dtype=np.int64)
    active = np.ones(n, dtype=bool)
    merges = np.zeros((max(n - 1, 0), 2), dtype=np.int64)
    heights = np.zeros(max(n - 1, 0), dtype=np.float64)
    iu = np.triu_indices(n, 1)
    for m in range(n - 1):
        # the best active pair: largest F, ties -> smallest (a, b) in row-major order
        act = active[iu[0]] & active[iu[1]]
        vals = S[iu][act]
        best = vals.max()
        rows, cols = iu[0][act], iu[1][act]
        k = np.flatnonzero(vals == best)[0]       # row-major order = lexicographic (a, b)
        a, b = int(rows[k]), int(cols[k])
        merges[m] = (a, b)
        heights[m] = (1.0 - float(best)) / 2.0
        na, nb = float(size[a]), float(size[b])
        for c in range(n):
            if not active[c] or c == a or c == b:
                continue
            v = (na * float(S[a, c]) + nb * float(S[b, c])) / float(size[a] + size[b])
            S[a, c] = S[c, a] = v
        size[a] += size[b]
        active[b] = False
    return merges, heights


def _neighbours(v: float):
    """The doubles just below and above v (finite v)."""
    return math.nextafter(v, -math.inf), math.nextafter(v, math.inf)


def cr_neg_log(x: float) -> float:
    """CR(-ln x) for a double x > 0: the double nearest the real value -ln x
    (ties to even; a double x != 1 has a transcendental log, so no real tie
    occurs).  Decimal ln at `prec` digits has error < 1 unit in the last
    digit; the result is accepted when the interval [approx - err, approx +
    err] rounds to one double, else the precision grows."""
    if x == 1.0:
        return 0.0
    prec = 60
    while True:
        with localcontext() as ctx:
            ctx.prec = prec
            approx = -(Decimal(x).ln())
            err = abs(approx) * Decimal(10) ** (-(prec - 2))
            lo, hi = approx - err, approx + err
        a, b = float(lo), float(hi)     # Decimal -> float is correctly rounded
        if a == b:
            return a
        prec *= 2


def dF_matrix(F: np.ndarray, delta: float = 0.02) -> np.ndarray:
    """d_ij = CR(-ln(RN(delta + F_ij))) off the diagonal, 0 on it (T4)."""
    n = F.shape[0]
    D = np.zeros((n, n), dtype=np.float64)
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i, j] = cr_neg_log(float(delta) + float(F[i, j]))
    return D


def upgma_distance(D: np.ndarray):
    """UPGMA on the symmetric distance matrix D (the diagonal is ignored): n - 1
    merges of the active pair (a, b), a < b, of smallest d, ties to the
    smallest (a, b); the merged cluster keeps id a; d(ab, c) = RN(RN(RN(n_a
    d_ac) + RN(n_b d_bc)) / (n_a + n_b)); height d_ab / 2."""
    n = D.shape[0]
    S = np.array(D, dtype=np.float64, copy=True)
    size = np.ones(n, dtype=np.int64)
    active = np.ones(n, dtype=bool)
    merges = np.zeros((max(n - 1, 0), 2), dtype=np.int64)
    heights = np.zeros(max(n - 1, 0), dtype=np.float64)
    iu = np.triu_indices(n, 1)
    for m in range(n - 1):
        act = active[iu[0]] & active[iu[1]]
        vals = S[iu][act]
        best = vals.min()
        rows, cols = iu[0][act], iu[1][act]
        k = np.flatnonzero(vals == best)[0]       # row-major order = lexicographic (a, b)
        a, b = int(rows[k]), int(cols[k])
        merges[m] = (a, b)
        heights[m] = float(best) / 2.0
        na, nb = float(size[a]), float(size[b])
        for c in range(n):
            if not active[c] or c == a or c == b:
                continue
            v = (na * float(S[a, c]) + nb * float(S[b, c])) / float(size[a] + size[b])
            S[a, c] = S[c, a] = v
        size[a] += size[b]
        active[b] = False
    return merges, heights


def upgma_dF(F: np.ndarray, delta: float = 0.02):
    """The d^F-form guide tree of a similarity matrix: upgma_distance(dF_matrix(F))."""
    return upgma_distance(dF_matrix(F, delta))
