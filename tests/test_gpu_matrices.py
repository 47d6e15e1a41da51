"""Full similarity matrices of every BASELINE config against the oracle.

S5 (the pairwise stage; Eq. 1): every bucket's full
numerator matrix C (uint16) and similarity matrix F (fp64) from the hot path
in the launch configuration bench.py times (HotPath.step: all buckets in one
sa_bucket_similarity_batch launch, padded rows) are hashed and compared with
the SHA-256 of the oracle's matrices for the same bucket (the oracle's own
partition), stored by scripts/make_golden_matrices.py, which calls only
oracle/.  S2d (Alg. 2 step 6): the full N x s numerator matrix of
every sequence against the global sample, written by the S2d GEMM epilogue
(sa_partition_debug.global_num), likewise.  Equal digests are equal matrices,
bit for bit (SURVEY §8(c) artifacts 2 and 6); on a mismatch the row-slab
digests name the slab that differs."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from paper_0905_1744_b200 import binding as B
from paper_0905_1744_b200.pipeline import HotPath
from sa_synth.generator import CONFIGS, generate

from .gpu_util import GOLDEN, load_golden, require_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    require_gpu()
    return B.Context()


def _golden_matrices(c):
    path = os.path.join(GOLDEN, f"matrices_cfg{c}.json")
    if not os.path.exists(path):
        pytest.skip(f"matrix digests for cfg{c} not generated")
    with open(path) as f:
        return json.load(f)


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _slabs(a: np.ndarray, slabs: int) -> list:
    n = a.shape[0]
    return [_sha(a[(s * n) // slabs:((s + 1) * n) // slabs]) for s in range(slabs)]


def _compare(name, a, want_sha, want_slabs, slabs):
    if _sha(a) == want_sha:
        return
    bad = [s for s, (x, y) in enumerate(zip(_slabs(a, slabs), want_slabs)) if x != y]
    pytest.fail(f"{name}: digest differs from the oracle's (row slabs {bad} of {slabs})")


@pytest.mark.parametrize("c", [1, 2, 3, 5, 4])
def test_s5_matrices_match_oracle(ctx, c):
    gm = _golden_matrices(c)
    g, _ = load_golden(c)
    cfg = CONFIGS[c]
    ds = generate(cfg)
    assert ds.sha256() == gm["dataset_sha256"]
    res, offs = to_dev(ds)
    hp = HotPath(ctx, cfg.p, cfg.samples_per_block)
    out = hp.step(res, offs, ds.n, 0)
    assert ctx.engine() == "tc"
    assert np.array_equal(out.part.bucket_of.cpu().numpy(), g["bucket_of"])
    gid = out.recv_global_idx.cpu().numpy()
    for (b, row, n_b), num, sim in zip(out.buckets, out.numerators, out.similarity):
        want = gm["buckets"][b]
        assert n_b == want["n"]
        assert np.array_equal(gid[row:row + n_b], np.flatnonzero(g["bucket_of"] == b))
        C = num.cpu().numpy()                       # n_b x n_b view of the padded rows
        _compare(f"cfg{c} bucket {b} C", C, want["C_sha256"], want["C_slabs"], gm["slabs"])
        del C
        F = sim.cpu().numpy()
        _compare(f"cfg{c} bucket {b} F", F, want["F_sha256"], want["F_slabs"], gm["slabs"])
        del F
    torch.cuda.empty_cache()


@pytest.mark.parametrize("c", [1, 2, 3, 5, 4])
def test_s2d_numerators_match_oracle(ctx, c):
    gm = _golden_matrices(c)
    g, _ = load_golden(c)
    cfg = CONFIGS[c]
    ds = generate(cfg)
    res, offs = to_dev(ds)
    P, nk = B.sa_kmer_profiles(ctx, res, offs)
    part = B.sa_partition(ctx, cfg.p, cfg.samples_per_block, P, nk, offs, 8000, ds.n, 0, debug=True,
                          want_global_num=True)
    assert np.array_equal(part.debug["sample_idx"].cpu().numpy(), g["sample_idx"])
    S2d = part.debug["global_num"].cpu().numpy()
    assert list(S2d.shape) == gm["s2d"]["shape"]
    if _sha(S2d) != gm["s2d"]["C_sha256"]:
        bounds = [(q * ds.n) // cfg.p for q in range(cfg.p + 1)]
        bad = [q for q in range(cfg.p) if _sha(S2d[bounds[q]:bounds[q + 1]]) != gm["s2d"]["block_sha256"][q]]
        pytest.fail(f"cfg{c} S2d numerators differ from the oracle's (blocks {bad})")
    # the keys of the same launch are the oracle's (stored digests)
    meta = json.load(open(os.path.join(GOLDEN, f"partition_cfg{c}.json")))
    gk = part.debug["global_key"].cpu().numpy().view(np.uint64).reshape(-1, 2)
    assert _sha(gk) == meta["global_key_sha256"]
