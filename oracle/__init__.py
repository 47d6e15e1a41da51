"""CPU oracle for the Sample-Align-D hot path (arxiv 0905.1744).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()``,
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs and
``scripts/make_golden.py`` may import or run anything here.  The product path
(``paper_0905_1744_b200``, ``libsa``) never imports it and shares no code,
headers, tables or constants with it.

Plain, slow, obviously correct: Python + numpy + ``fractions``, exact integers
everywhere the method is exact, fp64 only for the reported similarity / rank.
Each function cites the PAPER.md passage (``P:a-b``) or SPEC.md passage
(``S:a-b``) it follows; readings of silent or garbled passages are the SURVEY
§8(c) ids (Z1..Z21) listed in DESIGN.md §2.

Pins (tests/test_oracle.py, ``-m "not gpu"``):
  * kmer.count_kmers / kmer.profiles  -- brute-force substring enumeration,
    SPEC worked examples, total mass.
  * kmer.numerator / similarity       -- SPEC F = 2/3 example, F(X,X) = 1,
    symmetry, bounds, disjoint = 0, poly-residue closed form, containment.
  * kmer.rank_exact / rank_keys        -- SPEC pool examples re-derived for F
    (pool [X] -> 1, [X,Y] -> 5/6), brute-force ``Fraction`` sums, key bound.
  * partition.*                        -- SPEC position / pivot / bucket
    examples, closed-form partitions of identical sequences, two-cluster
    purity, permutation and 2N/p invariants.
  * tree.upgma (N4)                    -- SPEC guide-tree examples, the tie
    rule on all-tied matrices, scipy average-linkage heights, monotone heights.
No oracle function is "parity unpinned".
"""
