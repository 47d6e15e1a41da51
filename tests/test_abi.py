"""Host-side checks of the C ABI (-m "not gpu"): the library builds and loads,
exports every entry point include/sa.h declares, its pure-host routines
behave, and it refuses to compute without a GPU (no CPU fallback)."""
import os
import re
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_0905_1744_b200 import binding as B
from paper_0905_1744_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return B.load_library()


def declared_functions():
    with open(os.path.join(ROOT, "include", "sa.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sa_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ["sa_kmer_profiles", "sa_kmer_rank", "sa_partition", "sa_bucket_similarity", "sa_redistribute"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert names, "no declarations parsed"
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(B.EXPORTED) == names


def test_profile_stride(lib):
    assert B.sa_profile_stride(8000) == 8000
    assert B.sa_profile_stride(64) == 64
    assert B.sa_profile_stride(32) == 64
    assert B.sa_profile_stride(1) == 64
    assert B.sa_profile_stride(65536) == 65536


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_no_cpu_fallback(lib):
    with pytest.raises(B.SaError) as e:
        B.Context(0)
    assert e.value.status == B.SA_E_CUDA
    assert "no CPU fallback" in str(e.value)


def _V(C, nk, nkp):
    s = Fraction(0)
    for c, m in zip(C, nkp):
        d = min(nk, int(m))
        if d > 0:
            s += Fraction(int(c), d)
    return s


def test_exact_rank_compare_matches_fractions(lib):
    rng = np.random.default_rng(0)
    for trial in range(300):
        npool = int(rng.integers(1, 40))
        nkp = rng.integers(0, 60, size=npool)
        nka, nkb = int(rng.integers(0, 60)), int(rng.integers(0, 60))
        Ca = np.array([rng.integers(0, min(nka, m) + 1) for m in nkp], dtype=np.uint16)
        if trial % 3 == 0:
            nkb, Cb = nka, Ca.copy()                      # identical rows -> 0
        else:
            Cb = np.array([rng.integers(0, min(nkb, m) + 1) for m in nkp], dtype=np.uint16)
        want = _V(Ca, nka, nkp) - _V(Cb, nkb, nkp)
        sign = (want > 0) - (want < 0)
        assert B.sa_exact_rank_compare(Ca, nka, Cb, nkb, nkp) == sign


def test_exact_rank_compare_unequal_multisets_tie(lib):
    # 1/2 + 1/2 == 1/3 + 2/3 : equal rationals from different (C, D) terms
    nkp = np.array([2, 2, 3, 3], dtype=np.int32)
    Ca = np.array([1, 1, 0, 0], dtype=np.uint16)       # query nk 100 -> D = 2, 2, 3, 3
    Cb = np.array([0, 0, 1, 2], dtype=np.uint16)
    assert B.sa_exact_rank_compare(Ca, 100, Cb, 100, nkp) == 0
    Cb2 = np.array([0, 0, 1, 1], dtype=np.uint16)       # 2/3 < 1
    assert B.sa_exact_rank_compare(Ca, 100, Cb2, 100, nkp) == 1
    assert B.sa_exact_rank_compare(Cb2, 100, Ca, 100, nkp) == -1


def test_exact_rank_compare_large_lcm(lib):
    # many distinct denominators (lcm of 1..2000 has ~2900 bits); a tiny difference
    nkp = np.arange(1, 2001, dtype=np.int32)
    Ca = np.ones(2000, dtype=np.uint16)
    Cb = Ca.copy()
    Cb[1998] = 0
    Cb[1999] = 2          # 0/1999 + 2/2000 vs 1/1999 + 1/2000 : 1/2000 < 1/1999
    assert B.sa_exact_rank_compare(Ca, 5000, Cb, 5000, nkp) == 1
    assert B.sa_exact_rank_compare(Ca, 5000, Ca, 5000, nkp) == 0


def test_exchange_plan_host_logic():
    counts = np.array([[3, 1, 0, 2], [1, 1, 4, 0]], dtype=np.int64)   # 2 ranks x 4 buckets
    nbytes = counts * 100
    assert list(B.owned_buckets(4, 2, 0)) == [0, 1]
    assert list(B.owned_buckets(4, 2, 1)) == [2, 3]
    assert B.recv_sizes(counts, nbytes, 4, 2, 0) == (6, 600)
    assert B.recv_sizes(counts, nbytes, 4, 2, 1) == (6, 600)
    assert B.recv_sizes(counts[:1], nbytes[:1], 4, 1, 0) == (6, 600)


def test_host_checked_arguments_without_a_device(lib):
    """Argument errors are host-checked before any CUDA call (SA_E_INVAL with
    no GPU present); sa_last_error names the problem."""
    import ctypes
    # NULL context
    assert lib.sa_pack_upper_u16(None, None, 4, 4, None, None) == B.SA_E_INVAL
    assert b"ctx" in lib.sa_last_error()
    assert lib.sa_bucket_similarity_batch(None, 1, None, None, None, 8000, None, None, None, None) == B.SA_E_INVAL
    assert lib.sa_ctx_tc_operand(None) == -1
