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
the global best active pair.  Pins (tests/test_oracle.py): SPEC's examples
(1 sequence -> no merge; 2 -> one merge at (1 - F)/2; d(A,B) < d(A,C) =
d(B,C) -> (A, B) first), non-decreasing heights (UPGMA is monotone), and the
heights of scipy's average-linkage on 1 - F (a library routine) on tie-free
random matrices.
"""
from __future__ import annotations

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
