"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle against
something other than itself: SPEC/paper worked examples (tests/golden), brute
force enumeration, closed forms, exact ``Fraction`` arithmetic or invariants
the paper proves."""
import itertools
import math
import json
import os
from collections import Counter
from fractions import Fraction

import numpy as np
import pytest

from oracle import kmer, partition
from sa_synth.generator import ALPHABET, CONFIGS, from_sequences, generate


def codes(s):
    return [ALPHABET.index(c) for c in s]


@pytest.fixture(scope="module")
def spec(golden_dir):
    with open(os.path.join(golden_dir, "spec_examples.json")) as f:
        return json.load(f)


# ------------------------------------------------------------------ profiles
def test_count_kmers_spec_examples(spec):
    for ex in spec["count_kmers"]:
        got = kmer.count_kmers(codes(ex["seq"]), ex["k"])
        want = {tuple(codes(w)): c for w, c in ex["counts"].items()}
        assert got == want, ex["cite"]


def test_kmer_id_is_positional_numeral():
    # base-20 big-endian: (1, 2, 3) -> 1*400 + 2*20 + 3
    assert kmer.kmer_id((1, 2, 3), 20) == 443
    assert kmer.kmer_id((19, 19, 19), 20) == 7999
    assert kmer.kmer_id((1, 0), 2) == 2


@pytest.mark.parametrize("alphabet,k", [(2, 1), (2, 2), (2, 3), (3, 2), (3, 3)])
def test_profile_matches_exhaustive_enumeration(alphabet, k):
    """Exhaustive over every sequence of length <= 6: the dense bincount profile
    equals a hand enumeration of substrings, bin by bin."""
    for n in range(0, 7):
        for seq in itertools.product(range(alphabet), repeat=n):
            dense = kmer.profile(seq, k, alphabet)
            brute = Counter(tuple(seq[u:u + k]) for u in range(n - k + 1))
            want = np.zeros(alphabet ** k, dtype=np.int64)
            for w, c in brute.items():
                v = 0
                for r in w:
                    v = v * alphabet + r
                want[v] = c
            assert np.array_equal(dense, want), (seq, k)
            assert dense.sum() == max(0, n - k + 1)


def test_profiles_mass_and_dict_agreement():
    rng = np.random.default_rng(7)
    seqs = [rng.integers(0, 20, size=int(rng.integers(0, 60))) for _ in range(40)]
    ds = from_sequences(seqs)
    P, nk = kmer.profiles(ds.residues, ds.offsets, 3, 20)
    for i, s in enumerate(seqs):
        assert P[i].sum() == max(0, len(s) - 2) == nk[i]
        d = kmer.count_kmers(s, 3)
        for w, c in d.items():
            assert P[i, kmer.kmer_id(w, 20)] == c
        assert np.count_nonzero(P[i]) == len(d)


def test_profile_rejects_out_of_alphabet():
    with pytest.raises(ValueError):
        kmer.profile([0, 1, 20], 3, 20)


# ---------------------------------------------------------------- similarity
def _F(x, y, k, alphabet=20):
    cx = kmer.profile(codes(x), k, alphabet)
    cy = kmer.profile(codes(y), k, alphabet)
    return kmer.similarity(cx, cy, kmer.nkmers(len(x), k), kmer.nkmers(len(y), k))


def test_similarity_spec_examples(spec):
    for ex in spec["similarity"]:
        assert _F(ex["x"], ex["y"], ex["k"]) == Fraction(*ex["F"]), ex["cite"]


def _rand_seq(rng, lo, hi, alphabet=20):
    return rng.integers(0, alphabet, size=int(rng.integers(lo, hi + 1)))


def test_similarity_properties_random():
    rng = np.random.default_rng(11)
    for _ in range(200):
        alphabet = int(rng.integers(2, 21))
        x = _rand_seq(rng, 0, 40, alphabet)
        y = _rand_seq(rng, 0, 40, alphabet)
        cx, cy = kmer.profile(x, 3, alphabet), kmer.profile(y, 3, alphabet)
        nx, ny = kmer.nkmers(len(x), 3), kmer.nkmers(len(y), 3)
        c = kmer.numerator(cx, cy)
        d = kmer.denominator(nx, ny)
        # symmetry
        assert c == kmer.numerator(cy, cx)
        # brute-force multiset intersection size (independent of the dense path)
        bx, by = Counter(kmer.count_kmers(x, 3)), Counter(kmer.count_kmers(y, 3))
        assert c == sum((bx & by).values())
        # bounds 0 <= C <= D; equality iff the shorter multiset is contained
        assert 0 <= c <= max(d, 0)
        if d > 0:
            short, long_ = (bx, by) if nx <= ny else (by, bx)
            contained = all(long_[w] >= m for w, m in short.items())
            assert (c == d) == contained
        # self-similarity 1 when nk >= 1, 0 otherwise (Z4)
        assert kmer.similarity(cx, cx, nx, nx) == (1 if nx >= 1 else 0)


def test_similarity_closed_forms():
    # poly-residue: F(a^n, a^m) = 1 for n, m >= k
    for n, m in [(3, 3), (3, 50), (17, 9)]:
        assert _F("A" * n, "A" * m, 3) == 1
    # disjoint alphabets -> 0
    assert _F("ACDACDACD", "EFGHEFGH", 3) == 0
    # n < k -> 0 (Z4)
    assert _F("AC", "ACDEF", 3) == 0
    assert _F("AC", "AC", 3) == 0


def test_numerator_matrix_matches_pairwise():
    rng = np.random.default_rng(3)
    seqs = [_rand_seq(rng, 0, 80) for _ in range(23)]
    ds = from_sequences(seqs)
    P, nk = kmer.profiles(ds.residues, ds.offsets)
    C = kmer.numerator_matrix(P, P[:9])
    C4 = kmer.numerator_matrix(P, P[:9], workers=3)
    assert np.array_equal(C, C4)
    for i in range(len(seqs)):
        for j in range(9):
            bx, by = Counter(kmer.count_kmers(seqs[i], 3)), Counter(kmer.count_kmers(seqs[j], 3))
            assert C[i, j] == sum((bx & by).values())


# ---------------------------------------------------------------------- rank
def test_rank_spec_examples(spec):
    for ex in spec["rank"]:
        k = ex["k"]
        prof = [kmer.profile(codes(s), k, 20) for s in ex["pool"]]
        nks = [kmer.nkmers(len(s), k) for s in ex["pool"]]
        q = ex["query"]
        C = [kmer.numerator(prof[q], pj) for pj in prof]
        D = [kmer.denominator(nks[q], nj) for nj in nks]
        assert kmer.rank_exact(C, D) == Fraction(*ex["rank"]), ex["cite"]
        rs = kmer.RankSet(np.array([C]), np.array([D]))
        assert rs.fraction(0) == Fraction(*ex["rank"])


def test_rank_empty_pool_is_error():
    with pytest.raises(ValueError):
        kmer.rank_exact([], [])
    with pytest.raises(ValueError):
        kmer.RankSet(np.zeros((1, 0), dtype=np.int64), np.zeros((1, 0), dtype=np.int64))


def _brute_rank(C_row, D_row):
    s = Fraction(0)
    for c, d in zip(C_row, D_row):
        if d:
            s += Fraction(int(c), int(d))
    return s


def test_rankset_equals_fraction_sums_and_key_bound():
    """K_i / L equals the plain Fraction sum; the 64-bit fixed-point key obeys
    2^64 V - npool < key <= 2^64 V; orders agree with Fraction orders."""
    rng = np.random.default_rng(5)
    for trial in range(30):
        nq, npool = int(rng.integers(1, 12)), int(rng.integers(1, 15))
        nkq = rng.integers(0, 40, size=nq)
        nkp = rng.integers(0, 40, size=npool)
        D = kmer.denominator_matrix(nkq, nkp)
        C = (rng.random(D.shape) * (D + 1)).astype(np.int64)
        C = np.minimum(C, D)
        if trial % 3 == 0:      # force exact ties and C == D terms
            C[-1] = C[0]
            D[-1] = D[0]
            C[:, 0] = D[:, 0]
        rs = kmer.RankSet(C, D)
        V = [_brute_rank(C[i], D[i]) for i in range(nq)]
        for i in range(nq):
            assert Fraction(rs.K[i], rs.L) == V[i]
            assert rs.fraction(i) == V[i] / npool
            assert rs.f64(i) == float(V[i] / npool)
            key = rs.keys[i]
            assert V[i] * 2 ** 64 - npool < key <= V[i] * 2 ** 64
            direct = sum((int(c) << 64) // int(d) for c, d in zip(C[i], D[i]) if d)
            assert key == direct
        order_exact = sorted(range(nq), key=lambda i: (V[i], i))
        order_K = sorted(range(nq), key=lambda i: (rs.K[i], i))
        assert order_exact == order_K


# ----------------------------------------------------------------- partition
def test_partition_spec_examples(spec):
    for ex in spec["choose_local_samples"]:
        items = list(range(ex["n"]))
        assert partition.choose_local_samples(items, ex["count"]) == ex["positions"], ex["cite"]
    with pytest.raises(ValueError):
        partition.choose_local_samples([0, 1], 3)
    for ex in spec["select_pivots"]:
        assert partition.select_pivots(sorted(ex["Y"]), ex["p"]) == ex["pivots"], ex["cite"]
    for ex in spec["assign_buckets"]:
        assert partition.assign_bucket(ex["rank"], ex["pivots"]) == ex["bucket"], ex["cite"]


def test_block_bounds():
    assert partition.block_bounds(16, 4) == [0, 4, 8, 12, 16]
    assert partition.block_bounds(10, 3) == [0, 3, 6, 10]


def _identical(n, L=40, seed=0):
    rng = np.random.default_rng(seed)
    s = rng.integers(0, 20, size=L)
    ds = from_sequences([s] * n)
    return kmer.profiles(ds.residues, ds.offsets)


def test_partition_closed_form_identical_sequences(golden_dir):
    with open(os.path.join(golden_dir, "closed_form_partitions.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        P, nk = _identical(c["N"])
        r = partition.partition(P, nk, c["p"], c["samples_per_block"])
        assert r.pivots == c["pivots"]
        assert [len(b) for b in r.buckets] == c["sizes"]


def test_partition_two_clusters():
    """p = 2; cluster A = identical copies (F = 1 among them), cluster B =
    unrelated random sequences.  Global ranks of A exceed those of B, so bucket
    0 = B plus the lowest-index A member (the pivot itself: ties go to the lower
    bucket) and bucket 1 = the rest of A."""
    rng = np.random.default_rng(9)
    m = 20
    X = rng.integers(0, 20, size=120)
    seqs, isA = [], []
    for i in range(2 * m):
        if i % 2 == 0:
            seqs.append(X)
            isA.append(True)
        else:
            seqs.append(rng.integers(0, 20, size=120))
            isA.append(False)
    ds = from_sequences(seqs)
    P, nk = kmer.profiles(ds.residues, ds.offsets)
    r = partition.partition(P, nk, 2, 4)
    A = [i for i in range(2 * m) if isA[i]]
    B = [i for i in range(2 * m) if not isA[i]]
    assert r.pivots == [A[0]]
    assert sorted(r.buckets[0].tolist()) == sorted(B + [A[0]])
    assert sorted(r.buckets[1].tolist()) == A[1:]


def _check_invariants(r, n):
    allm = np.concatenate(r.buckets)
    assert np.array_equal(np.sort(allm), np.arange(n))           # permutation
    assert max(len(b) for b in r.buckets) <= 2 * n / r.p
    g = r.global_ranks
    pk = [(g.K[i], i) for i in r.pivots]
    for b, mem in enumerate(r.buckets):
        for i in mem.tolist():
            key = (g.K[i], i)
            if b < len(pk):
                assert key <= pk[b]
            if b > 0:
                assert key > pk[b - 1]


def test_partition_invariants_small_config():
    ds = generate(CONFIGS[1])
    P, nk = kmer.profiles(ds.residues, ds.offsets)
    r = partition.partition(P, nk, 4, 16)
    _check_invariants(r, ds.n)
    assert len(r.sample_idx) == 64 and len(set(r.sample_idx)) == 64
    assert len(r.candidates) == 12


def test_regular_sampling_load_bound_randomized():
    """1000 random rank distributions, N = 512, p = 4: no
    bucket exceeds 2N/p = 256 (the paper's regular-sampling bound)."""
    rng = np.random.default_rng(1)
    N, p = 512, 4
    w = N // p
    for t in range(1000):
        kind = t % 4
        if kind == 0:
            ranks = rng.random(N)
        elif kind == 1:
            ranks = np.sort(rng.random(N))                  # block-sorted skew
        elif kind == 2:
            ranks = rng.integers(0, 5, size=N).astype(float)  # heavy ties
        else:
            ranks = rng.lognormal(0, 3, size=N)
        keys = [(float(ranks[i]), i) for i in range(N)]
        Y = []
        for q in range(p):
            order = sorted(range(q * w, (q + 1) * w), key=lambda i: keys[i])
            Y.extend(partition.choose_local_samples(order, p - 1))
        Y = sorted(Y, key=lambda i: keys[i])
        piv = partition.select_pivots(Y, p)
        pk = [keys[i] for i in piv]
        sizes = Counter(partition.assign_bucket(keys[i], pk) for i in range(N))
        assert max(sizes.values()) <= 2 * N // p


def test_bucket_similarity_diagonal_symmetry():
    rng = np.random.default_rng(2)
    seqs = [_rand_seq(rng, 1, 50) for _ in range(15)]
    ds = from_sequences(seqs)
    P, nk = kmer.profiles(ds.residues, ds.offsets)
    C, F = partition.bucket_similarity(P, nk, np.arange(15))
    assert np.array_equal(C, C.T) and np.array_equal(F, F.T)
    for i in range(15):
        assert F[i, i] == (1.0 if nk[i] >= 1 else 0.0)
        for j in range(15):
            assert F[i, j] == float(kmer.similarity(P[i], P[j], nk[i], nk[j]))


# ------------------------------------------------- d^F rank ----
def test_dF_spec_examples():
    """SPEC S:124-126, S:133-134, S:141-143 with Delta = 0.02.  SPEC's
    hand-computed 0.37594 / 0.17807 carry a rounding slip of ~4e-5 (the exact
    values are 0.375906 / 0.178050), hence abs = 1e-4 on those two."""
    assert kmer.d_F(1.0) == pytest.approx(-0.01980, abs=5e-6)
    assert kmer.d_F(2 / 3) == pytest.approx(0.37594, abs=1e-4)
    assert kmer.d_F(0.0) == pytest.approx(3.91202, abs=5e-6)
    # pool [X, Y] with F(X,Y) = 2/3: R_X = (d(X,X) + d(X,Y)) / 2
    x, y = codes("ACAC"), codes("ACCA")
    px, py = kmer.profile(x, 2, 20), kmer.profile(y, 2, 20)
    C = np.array([[kmer.numerator(px, px), kmer.numerator(px, py)]])
    D = np.array([[3, 3]])
    assert kmer.RankSetDF(C, D).values[0] == pytest.approx(0.17807, abs=1e-4)
    # pool = [X]: -ln(1 + Delta); two disjoint samples: -ln(Delta)
    assert kmer.RankSetDF(np.array([[3]]), np.array([[3]])).values[0] == pytest.approx(-math.log(1.02), rel=1e-15)
    assert kmer.RankSetDF(np.array([[0, 0]]), np.array([[3, 5]])).values[0] == pytest.approx(-math.log(0.02),
                                                                                            rel=1e-15)


def test_dF_rank_is_mean_distance_and_order_reverses_monotone_case():
    """R^dF is the plain mean of -ln(Delta + F); when every F of one query
    dominates the other's term by term, its distance rank is smaller."""
    rng = np.random.default_rng(4)
    for _ in range(50):
        npool = int(rng.integers(1, 20))
        D = rng.integers(1, 40, size=(2, npool))
        C = np.minimum((rng.random((2, npool)) * (D + 1)).astype(np.int64), D)
        D[1] = D[0]
        C[1] = np.minimum(C[0] + rng.integers(0, 3, size=npool), D[0])   # F1 >= F0 termwise
        rs = kmer.RankSetDF(C, D)
        want = [sum(-math.log(0.02 + (c / d)) for c, d in zip(C[i], D[i])) / npool for i in range(2)]
        assert rs.values == pytest.approx(want, rel=1e-14)
        assert rs.values[1] <= rs.values[0]


def test_dF_partition_closed_form_and_invariants():
    with open(os.path.join(os.path.dirname(__file__), "golden", "closed_form_partitions.json")) as f:
        c = json.load(f)["cases"][1]
    P, nk = _identical(c["N"])
    r = partition.partition(P, nk, c["p"], c["samples_per_block"], rank_form="dF")
    assert r.pivots == c["pivots"] and [len(b) for b in r.buckets] == c["sizes"]
    ds = generate(CONFIGS[1])
    P, nk = kmer.profiles(ds.residues, ds.offsets)
    r = partition.partition(P, nk, 4, 16, rank_form="dF")
    allm = np.concatenate(r.buckets)
    assert np.array_equal(np.sort(allm), np.arange(ds.n))
    assert max(len(b) for b in r.buckets) <= 2 * ds.n / 4


# ------------------------------------------------------------ N4 tree ------
from oracle import tree  # noqa: E402


def test_upgma_spec_examples():
    """SPEC build_guide_tree examples, with d = 1 - F (reading T1):
    one sequence -> no merge; two -> one merge at half their distance; three
    with d(A,B) < d(A,C) = d(B,C) -> (A, B) merged first."""
    m, h = tree.upgma(np.ones((1, 1)))
    assert m.shape == (0, 2) and h.shape == (0,)
    F2 = np.array([[1.0, 0.3], [0.3, 1.0]])
    m, h = tree.upgma(F2)
    assert m.tolist() == [[0, 1]] and h[0] == (1.0 - 0.3) / 2.0
    F3 = np.array([[1.0, 0.8, 0.2], [0.8, 1.0, 0.2], [0.2, 0.2, 1.0]])
    m, h = tree.upgma(F3)
    assert m.tolist() == [[0, 1], [0, 2]]
    assert h.tolist() == [(1 - 0.8) / 2, (1 - 0.2) / 2]


def test_upgma_ties_take_the_smallest_pair():
    """All off-diagonal similarities equal: every average stays equal, so the
    tie rule alone orders the merges: (0,1), (0,2), (0,3), ..."""
    n = 6
    F = np.full((n, n), 0.25)
    np.fill_diagonal(F, 1.0)
    m, h = tree.upgma(F)
    assert m.tolist() == [[0, j] for j in range(1, n)]
    assert np.all(h == 0.375)


def test_upgma_matches_scipy_average_linkage():
    """UPGMA = average linkage: on tie-free random symmetric matrices the merge
    heights equal scipy's average-linkage heights on d = 1 - F (a library
    routine), and they never decrease."""
    from scipy.cluster.hierarchy import linkage
    from scipy.spatial.distance import squareform
    rng = np.random.default_rng(5)
    for n in (3, 7, 40):
        A = rng.random((n, n))
        F = (A + A.T) / 2
        np.fill_diagonal(F, 1.0)
        m, h = tree.upgma(F)
        D = 1.0 - F
        np.fill_diagonal(D, 0.0)
        Z = linkage(squareform(D, checks=False), method="average")
        assert np.allclose(h, Z[:, 2] / 2.0, rtol=0, atol=1e-12)
        assert np.all(np.diff(h) >= -1e-15)
        assert len(set(m[:, 1].tolist())) == n - 1 and np.all(m[:, 0] < m[:, 1])


# ----------------------------------------------------- N4 tree, d^F form ---
LN2_DIGITS = "0.693147180559945309417232121458176568075500134360255254120680"   # ln 2, 60 digits


def test_cr_neg_log_powers_of_two():
    """-ln(2^k) = -k ln 2: the correctly rounded double from the published
    digits of ln 2 (decimal multiplication, no log call) equals cr_neg_log."""
    from decimal import Decimal, localcontext
    for k in list(range(-60, 61)) + [-1000, 1000]:
        x = math.ldexp(1.0, k)
        with localcontext() as c:
            c.prec = 60
            want = float(-k * Decimal(LN2_DIGITS))
        assert tree.cr_neg_log(x) == want, k


def test_cr_neg_log_against_libm():
    """Within 1 ulp of libm's log everywhere (libm is not correctly rounded,
    so 1 ulp is the bound, not 0), exactly +0 at x = 1, and monotone."""
    rng = np.random.default_rng(11)
    xs = np.concatenate([rng.uniform(0.02, 1.02, 3000), [0.02, 1.0, 1.02, 0.5 + 2 ** -40]])
    prev = None
    for x in sorted(xs.tolist()):
        d = tree.cr_neg_log(x)
        ref = -math.log(x)
        assert abs(d - ref) <= math.ulp(ref) or d == ref, x
        if prev is not None:
            assert d <= prev
        prev = d
    assert math.copysign(1.0, tree.cr_neg_log(1.0)) == 1.0


def test_upgma_dF_spec_examples():
    """SPEC build_guide_tree in Eq. 2's distance: two sequences ->
    one merge at height d^F/2; d(A,B) < d(A,C) = d(B,C) -> (A, B) first; F = 1
    - Delta gives d = 0."""
    F2 = np.array([[1.0, 0.3], [0.3, 1.0]])
    m, h = tree.upgma_dF(F2, 0.02)
    assert m.tolist() == [[0, 1]] and h[0] == tree.cr_neg_log(0.32) / 2.0
    F3 = np.array([[1.0, 0.8, 0.2], [0.8, 1.0, 0.2], [0.2, 0.2, 1.0]])
    m, h = tree.upgma_dF(F3, 0.02)
    assert m.tolist() == [[0, 1], [0, 2]]
    d = tree.dF_matrix(np.array([[1.0, 0.98], [0.98, 1.0]]), 0.02)
    assert d[0, 1] == 0.0 and math.copysign(1.0, d[0, 1]) == 1.0


def test_upgma_distance_matches_scipy_average_linkage():
    """upgma_distance = average linkage: heights equal scipy's on the d^F matrix
    of tie-free random similarities; merge order follows the smallest d."""
    from scipy.cluster.hierarchy import linkage
    from scipy.spatial.distance import squareform
    rng = np.random.default_rng(6)
    for n in (3, 9, 30):
        A = rng.random((n, n))
        F = (A + A.T) / 2
        np.fill_diagonal(F, 1.0)
        D = tree.dF_matrix(F, 0.02)
        m, h = tree.upgma_distance(D)
        Z = linkage(squareform(D, checks=False), method="average")
        assert np.allclose(h, Z[:, 2] / 2.0, rtol=0, atol=1e-12)
        assert np.all(np.diff(h) >= -1e-15)
        # the d^F order reverses F's: on a 2-cluster matrix the same first merge as upgma(F)
        assert m[0].tolist() == tree.upgma(F)[0][0].tolist()
