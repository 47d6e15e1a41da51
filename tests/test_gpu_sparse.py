"""Parity of K2T's sparse layers >= 2 with the CPU oracle.

The tensor cores contract layer 1 only ([c >= 1], 8000 columns); every pair
that shares a bin both rows repeat gets the exact correction
min(c_i, c_j) - 1 from entries the GEMM epilogue adds (Eq. 1, P:264-269:
min(a, b) = [a >= 1][b >= 1] + (min(a, b) - 1)_+).  These tests force each
path (SA_K2T_SPARSE = 0 dense, 1 auto, 2 forced) on ragged sets that span
several tiles, with repeated 3-mers, duplicate rows, counts far above the 32
layers the dense path tracks, mixed sparse / dense problems in one launch,
and compare numerators, F and exact-rank keys bit for bit with the oracle."""
import numpy as np
import pytest
import torch

from oracle import kmer, partition
from paper_0905_1744_b200 import binding as B
from paper_0905_1744_b200.pipeline import HotPath
from sa_synth.generator import CONFIGS, from_sequences, generate

from .gpu_util import require_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    require_gpu()
    return B.Context()


def _rand_set(seed, n, lo=0, hi=420, alphabet=20, dup=0, runs=()):
    """Random sequences; `runs` = [(index, residue, length)] homopolymer runs
    prepended (a run of length L gives the bin of that residue's 3-mer the count L - 2)."""
    rng = np.random.default_rng(seed)
    seqs = [rng.integers(0, alphabet, size=int(rng.integers(lo, hi + 1))).astype(np.uint8) for _ in range(n)]
    for t in range(dup):
        seqs[(7 * t + 3) % n] = seqs[(11 * t) % n].copy()
    for i, r, L in runs:
        seqs[i] = np.concatenate([np.full(L, r, np.uint8), seqs[i]])
    return from_sequences(seqs)


def _oracle(ds):
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    Co, Fo = partition.bucket_similarity(Po, nko, np.arange(ds.n))
    return Po, nko, Co, Fo


def _check_all(ctx, P, nk, Co, Fo, nko, want_mode=None):
    n = nk.numel()
    num, sim = B.sa_bucket_similarity(ctx, P, nk)
    assert ctx.engine() == "tc"
    if want_mode is not None:
        assert [m for m, _ in ctx.tc_sparse()] == [want_mode]
    assert np.array_equal(num.cpu().numpy(), Co)
    assert np.array_equal(sim.cpu().numpy(), Fo)
    nums, sims = B.sa_bucket_similarity_batch(ctx, P, nk, [0, n], ld_align=16)
    assert np.array_equal(nums[0].cpu().numpy(), Co)
    assert np.array_equal(sims[0].cpu().numpy(), Fo)
    D = kmer.denominator_matrix(nko, nko)
    keys, _, _ = B.sa_kmer_rank(ctx, P, nk, P, nk)                    # symmetric keys
    assert ctx.engine() == "tc"
    assert B.keys_to_ints(keys) == kmer.RankSet(Co, D).keys
    if n < 2:
        return
    q = max(1, n // 3)
    keys, _, nm = B.sa_kmer_rank(ctx, P[:q], nk[:q], P[q:], nk[q:], want_numerators=True)   # rectangular
    assert ctx.engine() == "tc"
    if want_mode is not None:
        assert [m for m, _ in ctx.tc_sparse()] == [want_mode]
    assert np.array_equal(nm.cpu().numpy(), Co[:q, q:])
    assert B.keys_to_ints(keys) == kmer.RankSet(Co[:q, q:], D[:q, q:]).keys


@pytest.mark.parametrize("fp4,pair", [(1, 1), (1, 0), (0, 1)])
@pytest.mark.parametrize("n,hi,dup", [(600, 420, 0), (531, 3000, 40), (129, 60, 0), (256, 700, 9), (1, 50, 0),
                                      (2, 30, 0), (241, 400, 3)])
def test_sparse_forced_random(ctx, monkeypatch, n, hi, dup, fp4, pair):
    """Forced sparse layers: exact on every operand format, with and without
    CTA pairs, on sets from one row to several ragged tiles."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_SPARSE", "2")
    monkeypatch.setenv("SA_K2T_FP4", str(fp4))
    monkeypatch.setenv("SA_K2T_PAIR", str(pair))
    ds = _rand_set(9100 + n, n, 0, hi, dup=dup)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko, Co, Fo = _oracle(ds)
    _check_all(ctx, P, nk, Co, Fo, nko, want_mode=1)


@pytest.mark.parametrize("setting", ["0", "1", "2"])
def test_sparse_dense_auto_agree(ctx, monkeypatch, setting):
    """Dense, auto and forced sparse give the oracle's matrices and keys."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_SPARSE", setting)
    ds = _rand_set(77, 400, 30, 900, dup=6)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko, Co, Fo = _oracle(ds)
    _check_all(ctx, P, nk, Co, Fo, nko, want_mode={"0": 0, "2": 1}.get(setting))


@pytest.mark.parametrize("runs", [[(3, 4, 40), (77, 4, 38)],                  # counts 38, 36 (> 32 layers)
                                  [(0, 0, 300), (1, 0, 262), (5, 0, 282)],    # counts up to 298 (> 255)
                                  [(10, 13, 1200), (11, 13, 900), (12, 7, 2000)]])   # poly-Q / poly-I
def test_sparse_deep_counts_stay_on_tc(ctx, monkeypatch, runs):
    """Homopolymer runs (low-complexity repeats) give bin counts far above the
    32 threshold layers the dense path tracks and above the u8 SAD range: the
    sparse path keeps them on the tensor cores, exactly."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_SPARSE", "1")
    ds = _rand_set(81, 150, 3, 400, runs=runs)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko, Co, Fo = _oracle(ds)
    assert Po.max() > 32
    _check_all(ctx, P, nk, Co, Fo, nko, want_mode=1)


def test_sparse_mixed_batch(ctx, monkeypatch):
    """One launch over buckets of which some take the sparse path (short
    sequences) and some the dense one (long sequences whose 3-mers saturate:
    many terms per pair), plus empty and one-member buckets."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_SPARSE", "1")
    rng = np.random.default_rng(5)
    groups = [[rng.integers(0, 20, size=int(rng.integers(100, 400))) for _ in range(300)],
              [],
              [rng.integers(0, 20, size=200)],
              [rng.integers(0, 20, size=int(rng.integers(50, 600))) for _ in range(257)],
              [rng.integers(0, 20, size=int(rng.integers(1500, 2500))) for _ in range(90)]]
    seqs = [s.astype(np.uint8) for g in groups for s in g]
    ds = from_sequences(seqs)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    rb = np.cumsum([0] + [len(g) for g in groups]).tolist()
    nums, sims = B.sa_bucket_similarity_batch(ctx, P, nk, rb, ld_align=16)
    modes = [m for m, _ in ctx.tc_sparse()]
    assert modes == [1, 1, 1, 0]          # the empty bucket is skipped
    for b in range(len(groups)):
        if rb[b + 1] == rb[b]:
            continue
        Co, Fo = partition.bucket_similarity(Po, nko, np.arange(rb[b], rb[b + 1]))
        assert np.array_equal(nums[b].cpu().numpy(), Co), b
        assert np.array_equal(sims[b].cpu().numpy(), Fo), b


@pytest.mark.parametrize("c", [1, 2, 5])
def test_sparse_modes_on_configs(ctx, c):
    """Which path the BASELINE configs take (informative + exactness on the
    hot path): short-sequence configs go sparse, config 5's long sequences
    (k = 3 saturates: ~500 repeated bins per row) stay dense; the step's
    matrices equal the oracle's either way."""
    cfg = CONFIGS[c]
    ds = generate(cfg)
    res, offs = to_dev(ds)
    hp = HotPath(ctx, cfg.p, cfg.samples_per_block)
    out = hp.step(res, offs, ds.n, 0)
    modes = [m for m, _ in ctx.tc_sparse()]
    assert len(modes) == sum(1 for _, _, n in out.buckets if n > 0)
    if c in (1, 2):
        assert all(m == 1 for m in modes)
    if c == 5:
        assert all(m == 0 for m in modes)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    gid = out.recv_global_idx.cpu().numpy()
    for (b, r0, n_b), num, sim in zip(out.buckets, out.numerators, out.similarity):
        if n_b == 0:
            continue
        Co, Fo = partition.bucket_similarity(Po, nko, gid[r0:r0 + n_b])
        assert np.array_equal(num.cpu().numpy(), Co)
        assert np.array_equal(sim.cpu().numpy(), Fo)


def test_partition_with_poly_runs_matches_oracle(ctx, monkeypatch):
    """A config-2-shaped workload with low-complexity inserts (counts up to
    ~400 in one bin) partitions exactly like the oracle, its buckets' matrices
    included, without leaving the tensor cores."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    cfg = CONFIGS[2]
    base = generate(cfg)
    rng = np.random.default_rng(11)
    seqs = [base.seq(i).copy() for i in range(base.n)]
    for i in rng.choice(base.n, size=40, replace=False):
        L = int(rng.integers(35, 400))
        seqs[i] = np.concatenate([seqs[i][:50], np.full(L, 13, np.uint8), seqs[i][50:]])
    ds = from_sequences(seqs)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    assert Po.max() > 255
    part = B.sa_partition(ctx, cfg.p, cfg.samples_per_block, P, nk, offs, 8000, ds.n, 0, debug=True)
    assert ctx.engine() == "tc"
    ro = partition.partition(Po, nko, cfg.p, cfg.samples_per_block, workers=kmer.default_workers())
    assert np.array_equal(part.bucket_of.cpu().numpy(), ro.bucket_of)
    assert np.array_equal(part.debug["sample_idx"].cpu().numpy(), np.asarray(ro.sample_idx))
    hp = HotPath(ctx, cfg.p, cfg.samples_per_block)
    out = hp.step(res, offs, ds.n, 0)
    assert ctx.engine() == "tc"
    gid = out.recv_global_idx.cpu().numpy()
    for (b, r0, n_b), num, sim in zip(out.buckets, out.numerators, out.similarity):
        assert np.array_equal(gid[r0:r0 + n_b], ro.buckets[b])
        Co, Fo = partition.bucket_similarity(Po, nko, ro.buckets[b])
        assert np.array_equal(num.cpu().numpy(), Co)
        assert np.array_equal(sim.cpu().numpy(), Fo)
