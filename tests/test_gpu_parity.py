"""Parity of the CUDA path (libsa through the C ABI) with the CPU oracle.

Bit-exact for counts, numerators, keys (exact ranks), orders, samples,
pivots, buckets and redistributed sequences; fp64 similarities and ranks
within 1e-12 relative (BASELINE.json north_star) -- in practice equal.
Inputs are the seeded BASELINE.json workloads (sa_synth) and small seeded
adversarial sets."""
import numpy as np
import pytest
import torch

from oracle import kmer, partition
from paper_0905_1744_b200 import binding as B
from paper_0905_1744_b200.pipeline import HotPath, shard_range
from sa_synth.generator import CONFIGS, from_sequences, generate

from .gpu_util import assert_rel, digest, keys_u64, load_golden, prof_np, require_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    require_gpu()
    return B.Context()


@pytest.fixture(params=["auto", "sad", "u16", "u16imad"])
def engine(request, monkeypatch):
    """Run a test under each min-sum engine: auto runs the
    tensor-core threshold-layer engine (K2T) when the launch fits it, sad the
    uint8 SAD engine when every count is <= 255, u16 / u16imad force the
    uint16 VIMNMX engines."""
    monkeypatch.setenv("SA_ENGINE", request.param)
    return request.param


ENGINE_NAME = {"auto": "tc", "sad": "u8", "u16": "u16", "u16imad": "u16imad"}


def _rand_set(seed, n, lo=0, hi=420, alphabet=20, dup=0):
    rng = np.random.default_rng(seed)
    seqs = [rng.integers(0, alphabet, size=int(rng.integers(lo, hi + 1))) for _ in range(n)]
    for t in range(dup):                    # forced duplicates -> exact ties
        seqs[(7 * t + 3) % n] = seqs[(11 * t) % n].copy()
    return from_sequences(seqs)


# --------------------------------------------------------------- S1 ------
@pytest.mark.parametrize("c", [1, 2, 5])
def test_profiles_configs(ctx, c):
    ds = generate(CONFIGS[c])
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    assert np.array_equal(prof_np(P, 8000), Po)
    assert np.array_equal(nk.cpu().numpy(), nko)


@pytest.mark.parametrize("alphabet,k", [(20, 3), (4, 3), (2, 5), (20, 1), (3, 2), (4, 8)])
def test_profiles_small_alphabets_ragged(ctx, alphabet, k):
    """(4, 8): 65 536 bins, too many for two shared-memory rows -- the
    thread-store profiles_kernel runs instead of the bulk-copy one."""
    ds = _rand_set(alphabet * 10 + k, 77, 0, 60, alphabet)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs, k=k, alphabet=alphabet)
    bins = alphabet ** k
    Pn = P.cpu().numpy()
    Po, nko = kmer.profiles(ds.residues, ds.offsets, k, alphabet)
    assert np.array_equal(Pn[:, :bins], Po)
    assert not Pn[:, bins:].any()                 # padding to the 64-bin stride is zero
    assert np.array_equal(nk.cpu().numpy(), nko)  # includes n < k -> 0


def test_profiles_errors(ctx):
    """Argument errors are returned by the call; range errors are detected on
    the device and surface asynchronously (sa.h): at sa_ctx_check, or at
    sa_partition's count exchange -- with no host synchronisation in S1."""
    ds = from_sequences([np.array([0, 1, 2, 3], np.uint8), np.array([0, 20, 1, 2], np.uint8)])
    res, offs = to_dev(ds)
    B.sa_kmer_profiles(ctx, res, offs)          # enqueued, returns at once
    with pytest.raises(B.SaError) as e:
        ctx.check()
    assert e.value.status == B.SA_E_RANGE
    ctx.check()                                 # the flag was consumed
    with pytest.raises(B.SaError) as e:
        B.sa_kmer_profiles(ctx, res, offs, check=True)
    assert e.value.status == B.SA_E_RANGE
    P, nk = B.sa_kmer_profiles(ctx, res, offs)  # ... and sa_partition reports it at C3
    with pytest.raises(B.SaError) as e:
        B.sa_partition(ctx, 1, 1, P, nk, offs, 8000, 2, 0)
    assert e.value.status == B.SA_E_RANGE
    ctx.check()
    with pytest.raises(B.SaError) as e:
        B.sa_kmer_profiles(ctx, res, offs, k=0)
    assert e.value.status == B.SA_E_INVAL
    with pytest.raises(B.SaError) as e:
        B.sa_kmer_profiles(ctx, res, offs, k=4, alphabet=20)   # 160000 bins > 65536
    assert e.value.status == B.SA_E_INVAL
    # too many k-mers for uint16 counts
    big = from_sequences([np.zeros(65540, np.uint8)])
    r2, o2 = to_dev(big)
    with pytest.raises(B.SaError) as e:
        B.sa_kmer_profiles(ctx, r2, o2, check=True)
    assert e.value.status == B.SA_E_RANGE
    # empty set is a no-op
    P, nk = B.sa_kmer_profiles(ctx, torch.zeros(1, dtype=torch.uint8, device="cuda"),
                               torch.zeros(1, dtype=torch.int64, device="cuda"))
    assert P.shape[0] == 0 and nk.shape[0] == 0


def test_profiles_no_host_sync(ctx):
    """S1 never blocks the host (sa.h: range errors are sticky device flags,
    surfaced at ctx.check / C3): with the stream busy behind a ~0.5 s sleep
    kernel, sa_kmer_profiles returns while the stream is still busy, and its
    results are the oracle's once the stream drains."""
    ds = generate(CONFIGS[1])
    res, offs = to_dev(ds)
    B.sa_kmer_profiles(ctx, res, offs)      # one-time device setup happens here
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(1_000_000_000)    # ~0.5 s of device time ahead of S1
        P, nk = B.sa_kmer_profiles(ctx, res, offs, stream=s)
        busy = not s.query()
    assert busy, "sa_kmer_profiles waited for its stream"
    ctx.check(s)                            # the documented host block
    assert np.array_equal(nk.cpu().numpy(), kmer.profiles(ds.residues, ds.offsets)[1])


# --------------------------------------------------------------- S2 ------
@pytest.mark.parametrize("nq,npool,dup", [(300, 200, 0), (129, 257, 5), (1, 1, 0), (5, 700, 0)])
def test_kmer_rank_random(ctx, engine, nq, npool, dup):
    ds = _rand_set(nq * 1000 + npool, nq + npool, 0, 420, dup=dup)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    # the pool overlaps the queries (self terms present for the overlap)
    q0, p0 = 0, max(0, nq - npool // 3)
    keys, f64, num = B.sa_kmer_rank(ctx, P[q0:q0 + nq], nk[q0:q0 + nq], P[p0:p0 + npool], nk[p0:p0 + npool],
                                    want_numerators=True)
    C = kmer.numerator_matrix(Po[q0:q0 + nq], Po[p0:p0 + npool])
    D = kmer.denominator_matrix(nko[q0:q0 + nq], nko[p0:p0 + npool])
    assert np.array_equal(num.cpu().numpy(), C)
    rs = kmer.RankSet(C, D)
    got = B.keys_to_ints(keys)
    assert got == rs.keys
    assert_rel(f64.cpu().numpy(), [rs.f64(i) for i in range(nq)], 1e-12)


@pytest.mark.parametrize("n", [300, 129])
def test_kmer_rank_self_pool_symmetric_path(ctx, engine, n):
    """Pool = the queries themselves (upper-triangle tiles + column sums)."""
    ds = _rand_set(n + 5, n, 0, 420, dup=3)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    keys, f64, num = B.sa_kmer_rank(ctx, P, nk, P, nk, want_numerators=True)
    C = kmer.numerator_matrix(Po, Po)
    assert np.array_equal(num.cpu().numpy(), C)
    rs = kmer.RankSet(C, kmer.denominator_matrix(nko, nko))
    assert B.keys_to_ints(keys) == rs.keys
    assert_rel(f64.cpu().numpy(), [rs.f64(i) for i in range(n)], 1e-12)


def test_kmer_rank_empty_pool(ctx):
    P = torch.zeros((2, 8000), dtype=torch.uint16, device="cuda")
    nk = torch.ones(2, dtype=torch.int32, device="cuda")
    with pytest.raises(B.SaError) as e:
        B.sa_kmer_rank(ctx, P, nk, P[:0], nk[:0])
    assert e.value.status == B.SA_E_INVAL


# --------------------------------------------------------------- S5 ------
@pytest.mark.parametrize("n,dup,lo", [(300, 0, 0), (257, 20, 0), (128, 0, 2), (1, 0, 5), (2, 0, 0)])
def test_bucket_similarity_random(ctx, engine, n, dup, lo):
    ds = _rand_set(n * 7 + dup, n, lo, 420, dup=dup)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    num, sim = B.sa_bucket_similarity(ctx, P, nk)
    assert ctx.engine() == ENGINE_NAME[engine]
    Co, Fo = partition.bucket_similarity(Po, nko, np.arange(n))
    assert np.array_equal(num.cpu().numpy(), Co)
    s = sim.cpu().numpy()
    assert_rel(s, Fo, 1e-12)
    assert np.array_equal(s, Fo)     # one IEEE RN division on both sides


def test_f_division_free_is_ieee_rn(ctx):
    """The K2T matrix epilogue computes F = C/D as fma(r, RN(1/D), q0) with
    q0 = RN(C RN(1/D)) and r = C - q0 D (Markstein): bit-identical to IEEE RN
    division for every 0 <= C <= D <= 65535 (the whole domain of Eq. 1's F)."""
    assert B.selftest_f_division(0) == 0


@pytest.mark.parametrize("ld_align", [1, 16])
@pytest.mark.parametrize("sizes", [[0, 300, 1, 129, 0, 257], [2, 0, 0, 3]])
def test_bucket_similarity_batch(ctx, engine, sizes, ld_align):
    """sa_bucket_similarity_batch: every bucket of a ragged batch (empty ones
    included) equals the oracle's bucket matrices, in one engine launch; with
    padded rows (ld = n rounded up to 16) the padding columns stay untouched."""
    n = sum(sizes)
    ds = _rand_set(4242 + n, n, 0, 420, dup=3)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    rb = np.concatenate([[0], np.cumsum(sizes)])
    nums_in = [B.padded_matrix(sz, torch.uint16, "cuda", ld_align) if sz else None for sz in sizes]
    sims_in = [B.padded_matrix(sz, torch.float64, "cuda", ld_align) if sz else None for sz in sizes]
    for t in nums_in + sims_in:
        if t is not None:
            t.as_strided((t.shape[0], t.stride(0)), (t.stride(0), 1)).fill_(7)
    nums, sims = B.sa_bucket_similarity_batch(ctx, P, nk, rb, numerators=nums_in, similarity=sims_in)
    for t in nums + sims:
        if t is not None and t.stride(0) > t.shape[1]:
            pad = t.as_strided((t.shape[0], t.stride(0)), (t.stride(0), 1))[:, t.shape[1]:]
            assert bool((pad == 7).all()), "padding columns written"
    if n > 1:
        assert ctx.engine() == ENGINE_NAME[engine]
    for b, sz in enumerate(sizes):
        if sz == 0:
            assert nums[b] is None and sims[b] is None
            continue
        Co, Fo = partition.bucket_similarity(Po, nko, np.arange(rb[b], rb[b + 1]))
        assert np.array_equal(nums[b].cpu().numpy(), Co)
        assert np.array_equal(sims[b].cpu().numpy(), Fo)


@pytest.mark.parametrize("n,ld_align", [(0, 1), (1, 1), (257, 1), (300, 16)])
def test_pack_upper_u16(ctx, n, ld_align):
    """sa_pack_upper_u16: the packed upper triangle (diagonal included) of a
    bucket numerator matrix equals the row-major triu of the oracle's matrix."""
    ds = _rand_set(77 + n, n, 0, 420, dup=2) if n else None
    if n == 0:
        m = torch.empty((0, 0), dtype=torch.uint16, device="cuda")
        assert B.sa_pack_upper_u16(ctx, m).numel() == 0
        return
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    nums, _ = B.sa_bucket_similarity_batch(ctx, P, nk, [0, n], want_similarity=False, ld_align=ld_align)
    packed = B.sa_pack_upper_u16(ctx, nums[0]).cpu().numpy()
    Co, _ = partition.bucket_similarity(Po, nko, np.arange(n))
    assert np.array_equal(packed, Co[np.triu_indices(n)])


@pytest.mark.parametrize("grid", ["0", "1"])
@pytest.mark.parametrize("n,seed,ties", [(1, 0, False), (2, 1, False), (3, 2, False), (57, 3, False),
                                         (300, 4, False), (64, 5, True)])
def test_guide_tree_matches_oracle(ctx, monkeypatch, n, seed, ties, grid):
    """N4: sa_guide_tree on a bucket's S5 similarity matrix (random sets,
    duplicates -> exactly tied similarities) equals the oracle's UPGMA merge
    for merge and height for height (bit-exact fp64); both the one-CTA merge
    loop and the grid-wide cooperative one (SA_UPGMA_GRID)."""
    from oracle import tree
    monkeypatch.setenv("SA_UPGMA_GRID", grid)
    ds = _rand_set(600 + seed, n, 0, 420, dup=(n // 3 if ties else 0))
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    _, sims = B.sa_bucket_similarity_batch(ctx, P, nk, [0, n], want_numerators=False, ld_align=16)
    merges, heights = B.sa_guide_tree(ctx, sims[0])
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    _, Fo = partition.bucket_similarity(Po, nko, np.arange(n))
    mo, ho = tree.upgma(Fo)
    assert np.array_equal(merges.cpu().numpy().astype(np.int64), mo)
    assert np.array_equal(heights.cpu().numpy(), ho)


@pytest.mark.parametrize("c", [3, 4])
def test_guide_tree_grid_equals_one_cta_large(ctx, monkeypatch, c):
    """A 2 500-member bucket of config 3 / 4 sequences: the grid-wide merge
    loop and the one-CTA loop (identical IEEE operations and tie orders) build
    the same tree bit for bit."""
    ds = generate(CONFIGS[c]).subset(np.arange(2500))
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    _, sims = B.sa_bucket_similarity_batch(ctx, P, nk, [0, 2500], want_numerators=False, ld_align=16)
    out = {}
    for grid in ("0", "1"):
        monkeypatch.setenv("SA_UPGMA_GRID", grid)
        m, h = B.sa_guide_tree(ctx, sims[0])
        out[grid] = (m.cpu().numpy(), h.cpu().numpy())
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])
    assert np.all(np.diff(out["1"][1]) >= 0)


def test_guide_tree_batch_equals_single(ctx):
    """sa_guide_tree_batch: trees of mixed sizes (a grid-sized one, one-CTA
    sized ones, n = 2 and n = 1) built side by side in one launch equal the
    one-at-a-time trees bit for bit."""
    ds = generate(CONFIGS[3])
    sizes = [1800, 700, 130, 2, 1]
    res, offs = to_dev(ds.subset(np.arange(sum(sizes))))
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    bounds = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    _, sims = B.sa_bucket_similarity_batch(ctx, P, nk, bounds, want_numerators=False, ld_align=16)
    outs = B.sa_guide_tree_batch(ctx, sims)
    assert len(outs) == len(sizes)
    for sim, (m, h), n in zip(sims, outs, sizes):
        assert m.shape == (n - 1, 2) and h.shape == (n - 1,)
        m1, h1 = B.sa_guide_tree(ctx, sim)
        assert np.array_equal(m.cpu().numpy(), m1.cpu().numpy())
        assert np.array_equal(h.cpu().numpy(), h1.cpu().numpy())


@pytest.fixture
def dF_tree(ctx):
    ctx.set_tree_form(B.SA_TREE_DF, 0.02)
    yield ctx
    ctx.set_tree_form(B.SA_TREE_F)


def test_guide_tree_dF_log_values(dF_tree):
    """The d^F distance itself (reading T4): 2 x 2 trees, each one merge at
    height d/2, give the device's CR(-ln(RN(Delta + F))) for 2 000 random F
    and the edge values (F = 0, 1, 1 - Delta: d = +0) -- equal bit for bit to
    the oracle's decimal-certified rounding, none uncertified."""
    from oracle import tree
    ctx = dF_tree
    rng = np.random.default_rng(21)
    fs = np.concatenate([rng.random(2000), [0.0, 1.0, 0.98, 0.5, 0.25, 1e-9, 0.999999]])
    mats = []
    for f in fs:
        m = torch.full((2, 2), 1.0, dtype=torch.float64, device="cuda")
        m[0, 1] = m[1, 0] = float(f)
        mats.append(m)
    outs = B.sa_guide_tree_batch(ctx, mats)
    got = np.array([h.item() for _, h in outs])
    want = np.array([tree.cr_neg_log(0.02 + float(f)) / 2.0 for f in fs])
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, [(float(fs[i]), float(got[i]), float(want[i])) for i in bad[:8]]
    assert ctx.tree_uncertified() == 0


@pytest.mark.parametrize("grid", ["0", "1"])
def test_guide_tree_dF_matches_oracle(dF_tree, monkeypatch, grid):
    """N4 in Eq. 2's distance on config-1 bucket-sized and duplicate-holding
    sets: every merge and height equal to oracle.tree.upgma_dF (one-CTA and
    grid loops)."""
    from oracle import tree
    monkeypatch.setenv("SA_UPGMA_GRID", grid)
    ctx = dF_tree
    for n, dup in ((3, 0), (57, 0), (180, 6)):
        ds = _rand_set(1000 + n, n, 0, 300, dup=dup)
        res, offs = to_dev(ds)
        P, nk = B.sa_kmer_profiles(ctx, res, offs)
        _, sims = B.sa_bucket_similarity_batch(ctx, P, nk, [0, n], want_numerators=False, ld_align=16)
        m, h = B.sa_guide_tree(ctx, sims[0])
        mo, ho = tree.upgma_dF(sims[0].cpu().numpy(), 0.02)
        assert np.array_equal(m.cpu().numpy(), mo), n
        assert np.array_equal(h.cpu().numpy().view(np.uint64), ho.view(np.uint64)), n
        assert ctx.tree_uncertified() == 0


def test_guide_tree_on_a_config_bucket(ctx):
    """N4 on config 1's largest bucket after the full partition; the oracle
    side takes that bucket's members from the oracle's golden partition and
    its F from the oracle's own profiles."""
    from oracle import tree
    g, _ = load_golden(1)
    ds = generate(CONFIGS[1])
    res, offs = to_dev(ds)
    hp = HotPath(ctx, CONFIGS[1].p, CONFIGS[1].samples_per_block)
    out = hp.step(res, offs, ds.n, 0)
    sizes = [nb for _, _, nb in out.buckets]
    b = int(np.argmax(sizes))
    merges, heights = B.sa_guide_tree(ctx, out.similarity[b])
    members = np.flatnonzero(g["bucket_of"] == b)
    assert len(members) == sizes[b]
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    _, Fo = partition.bucket_similarity(Po, nko, members)
    mo, ho = tree.upgma(Fo)
    assert np.array_equal(merges.cpu().numpy().astype(np.int64), mo)
    assert np.array_equal(heights.cpu().numpy(), ho)
    assert np.all(np.diff(ho) >= 0)


def test_tc_falls_back_on_deep_counts(ctx, monkeypatch):
    """With the sparse layers off (SA_K2T_SPARSE=0), K2T tracks 32 threshold
    layers as MMA columns: a bin count of 33..255 must hand the call to the
    uint8 SAD engine on the device, exactly (with them on, the same set stays
    on K2T: tests/test_gpu_sparse.py)."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_SPARSE", "0")
    rng = np.random.default_rng(81)
    seqs = [rng.integers(0, 20, size=int(rng.integers(3, 400))) for _ in range(150)]
    seqs[3] = np.concatenate([np.full(40, 4, np.uint8), seqs[3]])     # 38 x EEE
    seqs[77] = np.concatenate([np.full(36, 4, np.uint8), seqs[77]])
    ds = from_sequences(seqs)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    assert 32 < Po.max() <= 255
    num, sim = B.sa_bucket_similarity(ctx, P, nk)
    assert ctx.engine() == "u8"
    Co, Fo = partition.bucket_similarity(Po, nko, np.arange(len(seqs)))
    assert np.array_equal(num.cpu().numpy(), Co)
    assert np.array_equal(sim.cpu().numpy(), Fo)


def test_tc_falls_back_on_column_overflow(ctx, monkeypatch):
    """Long sequences whose 3-mers repeat ~6 times keep more than 32768 layer
    columns: with the sparse layers off, K2T must decline and the SAD engine
    must run, exactly."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_SPARSE", "0")
    rng = np.random.default_rng(82)
    seqs = [rng.integers(0, 20, size=48000) for _ in range(3)] + \
        [rng.integers(0, 20, size=int(rng.integers(3, 400))) for _ in range(20)]
    ds = from_sequences(seqs)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    assert Po.max() <= 32
    num, sim = B.sa_bucket_similarity(ctx, P, nk)
    assert ctx.engine() == "u8"
    Co, Fo = partition.bucket_similarity(Po, nko, np.arange(len(seqs)))
    assert np.array_equal(num.cpu().numpy(), Co)
    assert np.array_equal(sim.cpu().numpy(), Fo)


@pytest.mark.parametrize("fp4,pair", [(1, 1), (1, 0), (0, 1), (0, 0)])
@pytest.mark.parametrize("n,hi,dup", [(600, 420, 0), (531, 3000, 40), (129, 60, 0), (256, 700, 9)])
def test_tc_layers_random(ctx, monkeypatch, n, hi, dup, fp4, pair):
    """K2T against the oracle on ragged sets that span several tiles (and a
    ragged CTA-pair half), with repeated 3-mers (several threshold layers) and
    duplicate rows; keys of the self-pool (symmetric: row + mirrored column
    sums) and of a rectangular pool, numerators and F; every operand format
    (e2m1 kind::mxf4 / u8 kind::i8) with and without CTA pairs (cta_group::2)."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_FP4", str(fp4))
    monkeypatch.setenv("SA_K2T_PAIR", str(pair))
    ds = _rand_set(9000 + n, n, 0, hi, dup=dup)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    num, sim = B.sa_bucket_similarity(ctx, P, nk)
    assert ctx.engine() == "tc"
    assert ctx.tc_operand() == ("e2m1" if fp4 else "u8")
    Co, Fo = partition.bucket_similarity(Po, nko, np.arange(n))
    assert np.array_equal(num.cpu().numpy(), Co)
    assert np.array_equal(sim.cpu().numpy(), Fo)
    nums, sims = B.sa_bucket_similarity_batch(ctx, P, nk, [0, n], ld_align=16)   # padded rows
    assert np.array_equal(nums[0].cpu().numpy(), Co)
    assert np.array_equal(sims[0].cpu().numpy(), Fo)
    D = kmer.denominator_matrix(nko, nko)
    keys, _, _ = B.sa_kmer_rank(ctx, P, nk, P, nk)
    assert ctx.engine() == "tc"
    assert B.keys_to_ints(keys) == kmer.RankSet(Co, D).keys
    q = n // 3
    keys, _, nm = B.sa_kmer_rank(ctx, P[:q], nk[:q], P[q:], nk[q:], want_numerators=True)
    assert ctx.engine() == "tc"
    assert np.array_equal(nm.cpu().numpy(), Co[:q, q:])
    assert B.keys_to_ints(keys) == kmer.RankSet(Co[:q, q:], D[:q, q:]).keys


def test_large_counts_fall_back_to_u16(ctx, monkeypatch):
    """A bin count above 255 (here 298 copies of AAA) cannot use the uint8
    SAD encoding; with the sparse layers off the auto engine must detect it
    and stay exact."""
    monkeypatch.setenv("SA_ENGINE", "auto")
    monkeypatch.setenv("SA_K2T_SPARSE", "0")
    rng = np.random.default_rng(8)
    seqs = [np.zeros(300, np.uint8), np.zeros(260, np.uint8)] + \
        [rng.integers(0, 20, size=int(rng.integers(3, 400))) for _ in range(140)]
    seqs[5] = np.concatenate([np.zeros(280, np.uint8), seqs[5]])
    ds = from_sequences(seqs)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    assert Po.max() > 255
    num, sim = B.sa_bucket_similarity(ctx, P, nk)
    assert ctx.engine() == "u16"
    Co, Fo = partition.bucket_similarity(Po, nko, np.arange(len(seqs)))
    assert np.array_equal(num.cpu().numpy(), Co)
    assert np.array_equal(sim.cpu().numpy(), Fo)
    keys, f64, nm = B.sa_kmer_rank(ctx, P[:50], nk[:50], P, nk, want_numerators=True)
    assert ctx.engine() == "u16"
    assert np.array_equal(nm.cpu().numpy(), Co[:50])
    assert B.keys_to_ints(keys) == kmer.RankSet(Co[:50], kmer.denominator_matrix(nko[:50], nko)).keys


# ----------------------------------------------------- S2-S3 partition ---
def _partition_g1(ctx, c):
    cfg = CONFIGS[c]
    ds = generate(cfg)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    part = B.sa_partition(ctx, cfg.p, cfg.samples_per_block, P, nk, offs, 8000, ds.n, 0, debug=True)
    return ds, P, nk, part


@pytest.mark.parametrize("c,eng", [(1, "auto"), (2, "auto"), (5, "auto"), (3, "auto"), (4, "auto"),
                                   (2, "u16"), (5, "u16imad")])
def test_partition_matches_golden(ctx, monkeypatch, c, eng):
    monkeypatch.setenv("SA_ENGINE", eng)
    g, meta = load_golden(c)
    ds, P, nk, part = _partition_g1(ctx, c)
    assert ds.sha256() == meta["dataset_sha256"]
    assert digest(prof_np(P, 8000)) == meta["profile_sha256"]          # S1 bit-exact at full size
    d = part.debug
    lk, gk = keys_u64(d["local_key"]), keys_u64(d["global_key"])
    assert digest(lk) == meta["local_key_sha256"]                       # S2a keys (exact ranks)
    assert digest(gk) == meta["global_key_sha256"]                      # S2d keys
    assert np.array_equal(d["local_order"].cpu().numpy(), g["local_order"])     # S2b
    assert np.array_equal(d["sample_idx"].cpu().numpy(), g["sample_idx"])       # S2b/S2c
    assert np.array_equal(d["global_order"].cpu().numpy(), g["global_order"])   # S3a
    assert np.array_equal(d["candidates"].cpu().numpy(), g["candidates"])       # S3b Y
    assert np.array_equal(B.pivot_global_idx(part.pivots).cpu().numpy(), g["pivots"])
    assert np.array_equal(part.bucket_of.cpu().numpy(), g["bucket_of"])         # S3c
    assert part.counts[0].tolist() == meta["bucket_sizes"]
    lf, gf = d["local_f64"].cpu().numpy(), d["global_f64"].cpu().numpy()
    if "local_f64" in g:
        assert_rel(lf, g["local_f64"])
        assert_rel(gf, g["global_f64"])
    else:
        idx = g["key_sample_idx"]
        assert_rel(lf[idx], g["local_f64_sample"])
        assert_rel(gf[idx], g["global_f64_sample"])
    assert part.exact_fallbacks == 0      # synthetic data has no uncertified comparisons


@pytest.mark.parametrize("segsort", ["grid", "cta"])
def test_partition_segment_sorts_agree(ctx, monkeypatch, segsort):
    """Both exact segment sorts (grid-wide passes, default; one CTA per block,
    SA_SEGSORT=cta) give the oracle's partition of config 2."""
    monkeypatch.setenv("SA_SEGSORT", segsort)
    g, meta = load_golden(2)
    ds, P, nk, part = _partition_g1(ctx, 2)
    d = part.debug
    assert np.array_equal(d["local_order"].cpu().numpy(), g["local_order"])
    assert np.array_equal(d["global_order"].cpu().numpy(), g["global_order"])
    assert np.array_equal(part.bucket_of.cpu().numpy(), g["bucket_of"])


def test_partition_invariants_any_size(ctx):
    """Properties that hold at any size: permutation, the
    regular-sampling bound 2N/p, pivot boundaries respected."""
    for c in (2, 5):
        ds, P, nk, part = _partition_g1(ctx, c)
        cfg = CONFIGS[c]
        b = part.bucket_of.cpu().numpy()
        assert b.min() >= 0 and b.max() < cfg.p
        sizes = np.bincount(b, minlength=cfg.p)
        assert sizes.sum() == ds.n and sizes.max() <= 2 * ds.n / cfg.p
        gk = [int(x) for x in B.keys_to_ints(part.debug["global_key"])]
        piv = B.pivot_global_idx(part.pivots).cpu().numpy()
        for i in range(ds.n):
            me = (gk[i], i)
            if b[i] < cfg.p - 1:
                assert me <= (gk[piv[b[i]]], int(piv[b[i]]))
            if b[i] > 0:
                assert me > (gk[piv[b[i] - 1]], int(piv[b[i] - 1]))


def test_partition_errors(ctx):
    ds = generate(CONFIGS[1])
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    with pytest.raises(B.SaError) as e:
        B.sa_partition(ctx, 4, 51, P, nk, offs, 8000, ds.n, 0)          # k_b > block size 50
    assert e.value.status == B.SA_E_INVAL
    with pytest.raises(B.SaError) as e:
        B.sa_partition(ctx, 0, 1, P, nk, offs, 8000, ds.n, 0)
    assert e.value.status == B.SA_E_INVAL


def test_partition_exact_path_duplicates(ctx):
    """Identical sequences have identical ranks: keys tie, the key order is
    not certified, and sa_partition resolves every such comparison exactly
    (big-integer rationals on the host); the result must equal the oracle's
    exact-rational partition, ties broken by index."""
    rng = np.random.default_rng(42)
    base = [rng.integers(0, 20, size=int(rng.integers(40, 300))) for _ in range(24)]
    seqs = [base[int(rng.integers(0, len(base)))].copy() for _ in range(96)]
    ds = from_sequences(seqs)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    part = B.sa_partition(ctx, 4, 6, P, nk, offs, 8000, ds.n, 0, debug=True)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    o = partition.partition(Po, nko, 4, 6)
    d = part.debug
    assert part.exact_fallbacks > 0
    assert B.keys_to_ints(d["local_key"]) == o.local_keys()
    assert B.keys_to_ints(d["global_key"]) == o.global_keys()
    assert d["local_order"].cpu().numpy().tolist() == [i for q in o.local_order for i in q]
    assert d["sample_idx"].cpu().numpy().tolist() == o.sample_idx
    assert d["global_order"].cpu().numpy().tolist() == [i for q in o.global_order for i in q]
    assert d["candidates"].cpu().numpy().tolist() == o.candidates
    assert B.pivot_global_idx(part.pivots).cpu().numpy().tolist() == o.pivots
    assert np.array_equal(part.bucket_of.cpu().numpy(), o.bucket_of)


def test_partition_identical_closed_form(ctx):
    """All sequences identical: the closed-form partition of
    tests/golden/closed_form_partitions.json (N = 200, p = 4)."""
    rng = np.random.default_rng(0)
    s = rng.integers(0, 20, size=40)
    ds = from_sequences([s] * 200)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    part = B.sa_partition(ctx, 4, 16, P, nk, offs, 8000, 200, 0)
    assert B.pivot_global_idx(part.pivots).cpu().numpy().tolist() == [25, 87, 162]
    assert part.counts[0].tolist() == [26, 62, 75, 37]


# ------------------------------------------------------- S4 + S5 (G=1) ---
@pytest.mark.parametrize("c", [1, 2])
def test_hot_path_step_matches_oracle(ctx, c):
    cfg = CONFIGS[c]
    ds = generate(cfg)
    res, offs = to_dev(ds)
    hp = HotPath(ctx, cfg.p, cfg.samples_per_block)
    out = hp.step(res, offs, ds.n, 0)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    o = partition.partition(Po, nko, cfg.p, cfg.samples_per_block)
    gid = out.recv_global_idx.cpu().numpy()
    assert np.array_equal(gid, np.concatenate(o.buckets))                 # S4 order (bucket, index)
    assert np.array_equal(out.recv_bucket.cpu().numpy(), o.bucket_of[gid])
    rr, ro = out.recv_residues.cpu().numpy(), out.recv_offsets.cpu().numpy()
    for j, i in enumerate(gid):
        assert np.array_equal(rr[ro[j]:ro[j + 1]], ds.seq(int(i)))
    for (b, row, n_b), num, sim in zip(out.buckets, out.numerators, out.similarity):
        Co, Fo = partition.bucket_similarity(Po, nko, o.buckets[b])
        assert np.array_equal(num.cpu().numpy(), Co)
        assert np.array_equal(sim.cpu().numpy(), Fo)


def test_hot_path_full_size_sampled(ctx):
    """Config 4 at full size, in the launch configuration bench.py times:
    sampled rows of every bucket's matrices against the oracle, computed one
    row at a time; symmetry and unit diagonal on a sampled block."""
    cfg = CONFIGS[4]
    g, meta = load_golden(4)
    ds = generate(cfg)
    res, offs = to_dev(ds)
    hp = HotPath(ctx, cfg.p, cfg.samples_per_block)
    out = hp.step(res, offs, ds.n, 0)
    assert np.array_equal(out.part.bucket_of.cpu().numpy(), g["bucket_of"])
    gid = out.recv_global_idx.cpu().numpy()
    rng = np.random.default_rng(4)
    for (b, row, n_b), num, sim in zip(out.buckets, out.numerators, out.similarity):
        members = gid[row:row + n_b]
        assert np.array_equal(members, np.flatnonzero(g["bucket_of"] == b))
        Pm, nkm = kmer.profiles(ds.subset(members).residues, ds.subset(members).offsets)
        for r in list(rng.choice(n_b, size=3, replace=False)) + [n_b - 1]:
            Crow = kmer.numerator_matrix(Pm[r:r + 1], Pm)[0]
            Drow = np.minimum(nkm[r], nkm)
            assert np.array_equal(num[r].cpu().numpy(), Crow)
            Frow = np.where(Drow > 0, Crow / np.maximum(Drow, 1), 0.0)
            assert np.array_equal(sim[r].cpu().numpy(), Frow)
        blk = num[:200, :200].cpu().numpy()
        assert np.array_equal(blk, blk.T)
        assert np.all(np.diag(sim[:200, :200].cpu().numpy()) == 1.0)


# ------------------------------------------------- d^F rank ----
def _close(a, b, tol=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b))), np.max(np.abs(a - b))


@pytest.mark.parametrize("nq,npool", [(300, 200), (5, 700)])
def test_kmer_rank_dF_form(ctx, engine, nq, npool):
    ds = _rand_set(nq * 31 + npool, nq + npool, 0, 420, dup=2)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    p0 = max(0, nq - npool // 3)
    ctx.set_rank_form(B.SA_RANK_DF, 0.02)
    try:
        keys, f64, _ = B.sa_kmer_rank(ctx, P[:nq], nk[:nq], P[p0:p0 + npool], nk[p0:p0 + npool])
    finally:
        ctx.set_rank_form(B.SA_RANK_F)
    C = kmer.numerator_matrix(Po[:nq], Po[p0:p0 + npool])
    rs = kmer.RankSetDF(C, kmer.denominator_matrix(nko[:nq], nko[p0:p0 + npool]), 0.02)
    _close(f64.cpu().numpy(), rs.values)


def test_rank_form_errors(ctx):
    with pytest.raises(B.SaError):
        ctx.set_rank_form(7)
    with pytest.raises(B.SaError):
        ctx.set_rank_form(B.SA_RANK_DF, 0.0)


@pytest.mark.parametrize("c", [1, 2, 5])
def test_partition_dF_matches_oracle(ctx, c):
    """The paper's own distance rank (Eq. 2-3): orders, samples, pivots and
    buckets equal the oracle's wherever the fp64 window certifies them (here:
    everywhere, `uncertified == 0`); ranks within 1e-12."""
    cfg = CONFIGS[c]
    ds = generate(cfg)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    ctx.set_rank_form(B.SA_RANK_DF, 0.02)
    try:
        part = B.sa_partition(ctx, cfg.p, cfg.samples_per_block, P, nk, offs, 8000, ds.n, 0, debug=True)
    finally:
        ctx.set_rank_form(B.SA_RANK_F)
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    o = partition.partition(Po, nko, cfg.p, cfg.samples_per_block, workers=kmer.default_workers(), rank_form="dF")
    d = part.debug
    assert part.uncertified == 0
    _close(d["local_f64"].cpu().numpy(), o.local_f64())
    _close(d["global_f64"].cpu().numpy(), o.global_f64())
    assert d["local_order"].cpu().numpy().tolist() == [i for q in o.local_order for i in q]
    assert d["sample_idx"].cpu().numpy().tolist() == o.sample_idx
    assert d["global_order"].cpu().numpy().tolist() == [i for q in o.global_order for i in q]
    assert d["candidates"].cpu().numpy().tolist() == o.candidates
    assert B.pivot_global_idx(part.pivots).cpu().numpy().tolist() == o.pivots
    assert np.array_equal(part.bucket_of.cpu().numpy(), o.bucket_of)
