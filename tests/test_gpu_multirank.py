"""Multi-rank path of sa_partition / sa_redistribute / S5 on ONE GPU: G ranks
as threads with their own sa_ctx and a host-barrier communicator
(tests/threadcomm.py).  Results must not depend on G: the
partition of G ranks equals the single-rank partition and the oracle's."""
import numpy as np
import pytest
import torch

from paper_0905_1744_b200 import binding as B
from paper_0905_1744_b200.pipeline import HotPath, shard_range
from sa_synth.generator import CONFIGS, generate

from .gpu_util import load_golden, require_gpu
from .threadcomm import run_ranks

pytestmark = pytest.mark.gpu


def _run(G, cfg, ds):
    def fn(rank, ctx):
        first, last = shard_range(ds.n, cfg.p, G, rank)
        r0, r1 = int(ds.offsets[first]), int(ds.offsets[last])
        res = torch.from_numpy(ds.residues[r0:r1].copy()).cuda()
        offs = torch.from_numpy(ds.offsets[first:last + 1] - ds.offsets[first]).cuda()
        out = HotPath(ctx, cfg.p, cfg.samples_per_block).step(res, offs, ds.n, first, debug=True)
        torch.cuda.synchronize()
        return {
            "first": first,
            "bucket_of": out.part.bucket_of.cpu().numpy(),
            "pivots": B.pivot_global_idx(out.part.pivots).cpu().numpy(),
            "counts": out.part.counts.copy(),
            "gid": out.recv_global_idx.cpu().numpy(),
            "bkt": out.recv_bucket.cpu().numpy(),
            "res": out.recv_residues.cpu().numpy(), "offs": out.recv_offsets.cpu().numpy(),
            "sample_idx": out.part.debug["sample_idx"].cpu().numpy(),
            "candidates": out.part.debug["candidates"].cpu().numpy(),
            "num": [(b, n, x.view(torch.int16).cpu().numpy().view(np.uint16) if x is not None else None)
                    for (b, _, n), x in zip(out.buckets, out.numerators)],
            "sim": [x.cpu().numpy() if x is not None else None for x in out.similarity],
        }
    return run_ranks(G, fn)


@pytest.mark.parametrize("n,p,kb,Gs", [(1003, 6, 7, (1, 2, 3, 6)), (203, 3, 5, (1, 3)), (97, 1, 4, (1,))])
def test_ragged_blocks_odd_p_match_oracle(n, p, kb, Gs):
    """N not divisible by p (blocks of unequal size, Z13), odd p (pivot index
    floor(p/2) + jp, Z9), p = 1 (one bucket): every rank count gives the
    oracle's partition and buckets."""
    require_gpu()
    from oracle import kmer, partition
    from sa_synth.generator import WorkloadConfig
    cfg = WorkloadConfig("ragged", n, 1, ("uniform", 30, 400), 0.3, 0.05, p, kb, 11)   # p, k_b for HotPath
    ds = _mixed(n, seed=11)
    P, nk = kmer.profiles(ds.residues, ds.offsets)
    o = partition.partition(P, nk, p, kb)
    for G in Gs:
        outs = _run(G, cfg, ds)
        assert np.array_equal(np.concatenate([x["bucket_of"] for x in outs]), o.bucket_of), G
        assert np.array_equal(np.concatenate([x["gid"] for x in outs]), np.concatenate(o.buckets)), G
        for x in outs:
            assert x["pivots"].tolist() == o.pivots
            assert x["candidates"].tolist() == o.candidates and x["sample_idx"].tolist() == o.sample_idx


def _mixed(n, seed):
    """n sequences from a few random families (lengths 30..400), seeded."""
    from sa_synth.generator import from_sequences
    rng = np.random.default_rng(seed)
    anc = [rng.integers(0, 20, size=int(rng.integers(30, 400))) for _ in range(7)]
    seqs = []
    for i in range(n):
        a = anc[int(rng.integers(0, 7))].copy()
        m = rng.random(a.shape[0]) < 0.3
        a[m] = rng.integers(0, 20, size=int(m.sum()))
        seqs.append(a)
    return from_sequences(seqs)


@pytest.mark.parametrize("c,Gs", [(2, (2, 4, 8)), (1, (2, 4))])
def test_rank_count_invariance(c, Gs):
    require_gpu()
    cfg = CONFIGS[c]
    ds = generate(cfg)
    g, meta = load_golden(c)
    ref = _run(1, cfg, ds)[0]
    assert np.array_equal(ref["bucket_of"], g["bucket_of"])
    for G in Gs:
        outs = _run(G, cfg, ds)
        bucket_of = np.concatenate([o["bucket_of"] for o in outs])
        assert np.array_equal(bucket_of, g["bucket_of"]), G                 # S3c, every rank's shard
        for o in outs:
            assert np.array_equal(o["pivots"], g["pivots"])                 # identical pivots everywhere (O2)
            assert np.array_equal(o["sample_idx"], g["sample_idx"])         # S2c allgather order
            assert np.array_equal(o["candidates"], g["candidates"])         # S3b allgather order
            assert np.array_equal(o["counts"], outs[0]["counts"])           # C3 matrix
        # S4: rank r holds its buckets in (bucket, global id) order, residues intact
        gid = np.concatenate([o["gid"] for o in outs])
        assert np.array_equal(gid, ref["gid"])
        assert np.array_equal(np.concatenate([o["bkt"] for o in outs]), ref["bkt"])
        for o in outs:
            for j, i in enumerate(o["gid"]):
                assert np.array_equal(o["res"][o["offs"][j]:o["offs"][j + 1]], ds.seq(int(i)))
        # S5 matrices identical to the single-rank run
        ref_num = {b: x for b, n, x in ref["num"]}
        ref_sim = {b: x for (b, n, _), x in zip(ref["num"], ref["sim"])}
        for o in outs:
            for (b, n, x), s in zip(o["num"], o["sim"]):
                assert np.array_equal(x, ref_num[b]) and np.array_equal(s, ref_sim[b])


def test_nccl_communicator_one_rank_matches():
    """The torch.distributed / NCCL communicator (TorchComm) driven by libsa's
    callbacks on a 1-rank NCCL group: every collective of sa_partition and
    sa_redistribute goes through all_gather_into_tensor / all_to_all_single on
    raw device buffers and the caller's stream; results equal the golden."""
    require_gpu()
    import socket

    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cfg = CONFIGS[2]
    ds = generate(cfg)
    g, meta = load_golden(2)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        ctx = B.Context(0)
        comm = B.TorchComm(device="cuda")
        ctx.attach_comm(comm)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            res = torch.from_numpy(ds.residues.copy()).cuda()
            offs = torch.from_numpy(ds.offsets.copy()).cuda()
            out = HotPath(ctx, cfg.p, cfg.samples_per_block).step(res, offs, ds.n, 0, debug=True)
        torch.cuda.synchronize()
        assert not comm.errors, comm.errors
        assert np.array_equal(out.part.bucket_of.cpu().numpy(), g["bucket_of"])
        assert np.array_equal(out.part.debug["sample_idx"].cpu().numpy(), g["sample_idx"])
        assert np.array_equal(out.part.debug["candidates"].cpu().numpy(), g["candidates"])
        gid = out.recv_global_idx.cpu().numpy()
        assert np.array_equal(gid, np.concatenate([np.flatnonzero(g["bucket_of"] == b) for b in range(cfg.p)]))
        rr, ro = out.recv_residues.cpu().numpy(), out.recv_offsets.cpu().numpy()
        for j in range(0, len(gid), 97):
            assert np.array_equal(rr[ro[j]:ro[j + 1]], ds.seq(int(gid[j])))
    finally:
        dist.destroy_process_group()


def test_libsa_nccl_communicator_one_rank():
    """libsa's own NCCL communicator (sa_nccl_unique_id / sa_ctx_attach_nccl):
    a 1-rank group, so every exchange of sa_partition (ncclAllGather) and
    sa_redistribute (the packed all-to-all path, its own block by device copy)
    runs through NCCL on the caller's stream with no Python in between; the
    artifacts equal the golden partition.  (Two ranks need two GPUs.)"""
    require_gpu()
    cfg = CONFIGS[2]
    ds = generate(cfg)
    g, meta = load_golden(2)
    ctx = B.Context(0)
    ctx.attach_nccl(B.nccl_unique_id(), 1, 0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        res = torch.from_numpy(ds.residues.copy()).cuda()
        offs = torch.from_numpy(ds.offsets.copy()).cuda()
        out = HotPath(ctx, cfg.p, cfg.samples_per_block).step(res, offs, ds.n, 0, debug=True)
    torch.cuda.synchronize()
    ctx.check()
    assert np.array_equal(out.part.bucket_of.cpu().numpy(), g["bucket_of"])
    assert np.array_equal(out.part.debug["sample_idx"].cpu().numpy(), g["sample_idx"])
    gid = out.recv_global_idx.cpu().numpy()
    assert np.array_equal(gid, np.concatenate([np.flatnonzero(g["bucket_of"] == b) for b in range(cfg.p)]))
    rr, ro = out.recv_residues.cpu().numpy(), out.recv_offsets.cpu().numpy()
    for j in range(0, len(gid), 97):
        assert np.array_equal(rr[ro[j]:ro[j + 1]], ds.seq(int(gid[j])))
    with pytest.raises(B.SaError) as e:
        ctx.attach_nccl(B.nccl_unique_id(), 1, 0)
    assert e.value.status == B.SA_E_STATE
