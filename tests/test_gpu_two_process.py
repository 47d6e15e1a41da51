"""The multi-process path of libsa on one GPU: two processes (spawned), each
with its own context and a world-size-2 gloo process group whose collectives
stage the device buffers through host memory (TorchComm(stage_host=True)), so
no kernel of one process waits on the other's.  Each rank runs HotPath.step
on its shard of config 2 -- sa_partition (C1-C3 allgathers), sa_redistribute
(C4 all-to-all) and the S5 matrices of the buckets it owns -- and every
artifact is compared with the single-rank run and with the oracle (golden
partition, oracle bucket matrices).  Algorithm 2; the
decomposition the paper distributes over processors."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from .gpu_util import load_golden, require_gpu

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, c, q):
    try:
        import torch.distributed as dist

        from paper_0905_1744_b200 import binding as B
        from paper_0905_1744_b200.pipeline import HotPath, shard_range
        from sa_synth.generator import CONFIGS, generate
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        cfg = CONFIGS[c]
        ds = generate(cfg)
        first, last = shard_range(ds.n, cfg.p, world, rank)
        r0, r1 = int(ds.offsets[first]), int(ds.offsets[last])
        res = torch.from_numpy(ds.residues[r0:r1].copy()).cuda()
        offs = torch.from_numpy(ds.offsets[first:last + 1] - ds.offsets[first]).cuda()
        ctx = B.Context(0)
        comm = B.TorchComm(device="cuda", stage_host=True)
        ctx.attach_comm(comm)
        out = HotPath(ctx, cfg.p, cfg.samples_per_block).step(res, offs, ds.n, first, debug=True)
        torch.cuda.synchronize()
        ctx.check()
        d = out.part.debug
        q.put({"rank": rank, "first": first, "errors": list(comm.errors),
               "bucket_of": out.part.bucket_of.cpu().numpy(), "counts": out.part.counts,
               "sample_idx": d["sample_idx"].cpu().numpy(), "candidates": d["candidates"].cpu().numpy(),
               "local_key": d["local_key"].cpu().numpy(), "global_key": d["global_key"].cpu().numpy(),
               "local_order": d["local_order"].cpu().numpy(), "global_order": d["global_order"].cpu().numpy(),
               "gid": out.recv_global_idx.cpu().numpy(), "res": out.recv_residues.cpu().numpy(),
               "offs": out.recv_offsets.cpu().numpy(),
               "mats": [(b, n, num.cpu().numpy(), sim.cpu().numpy()) for (b, _, n), num, sim in
                        zip(out.buckets, out.numerators, out.similarity) if n > 0]})
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put({"rank": rank, "fatal": repr(e) + traceback.format_exc()})


@pytest.mark.parametrize("c", [2])
def test_two_processes_match_single_rank_and_oracle(c):
    require_gpu()
    from oracle import kmer, partition
    from paper_0905_1744_b200 import binding as B
    from paper_0905_1744_b200.pipeline import HotPath
    from sa_synth.generator import CONFIGS, generate
    cfg = CONFIGS[c]
    ds = generate(cfg)
    g, meta = load_golden(c)
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_rank_main, args=(r, 2, port, c, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=600) for _ in procs], key=lambda o: o["rank"])
    for p in procs:
        p.join(timeout=120)
    for o in outs:
        assert "fatal" not in o, o.get("fatal")
        assert not o["errors"], o["errors"]
    # single-rank reference run in this process
    ctx = B.Context(0)
    res = torch.from_numpy(ds.residues.copy()).cuda()
    offs = torch.from_numpy(ds.offsets.copy()).cuda()
    ref = HotPath(ctx, cfg.p, cfg.samples_per_block).step(res, offs, ds.n, 0, debug=True)
    rd = ref.part.debug
    # S2-S3: shards concatenate to the single-rank artifacts and the oracle's
    cat = lambda k: np.concatenate([o[k] for o in outs])   # noqa: E731
    assert np.array_equal(cat("bucket_of"), g["bucket_of"])
    assert np.array_equal(cat("bucket_of"), ref.part.bucket_of.cpu().numpy())
    for k in ("local_key", "global_key", "local_order", "global_order"):
        assert np.array_equal(cat(k), rd[k].cpu().numpy()), k
    assert np.array_equal(cat("local_order"), g["local_order"])
    assert np.array_equal(cat("global_order"), g["global_order"])
    for o in outs:   # replicated artifacts: identical on both ranks
        assert np.array_equal(o["sample_idx"], g["sample_idx"])
        assert np.array_equal(o["candidates"], g["candidates"])
        assert np.array_equal(o["counts"], outs[0]["counts"])
    # S4: every rank received exactly its buckets' members, in (bucket, index) order, with their residues
    pb = cfg.p // 2
    for o in outs:
        want = np.concatenate([np.flatnonzero(g["bucket_of"] == b) for b in range(o["rank"] * pb, (o["rank"] + 1) * pb)])
        assert np.array_equal(o["gid"], want)
        for j, i in enumerate(o["gid"]):
            assert np.array_equal(o["res"][o["offs"][j]:o["offs"][j + 1]], ds.seq(int(i)))
    # S5: the owned buckets' matrices equal the single-rank run's and the oracle's
    Po, nko = kmer.profiles(ds.residues, ds.offsets)
    ref_m = {b: (num.cpu().numpy(), sim.cpu().numpy()) for (b, _, n), num, sim in
             zip(ref.buckets, ref.numerators, ref.similarity) if n > 0}
    seen = set()
    for o in outs:
        for b, n, num, sim in o["mats"]:
            assert np.array_equal(num, ref_m[b][0]) and np.array_equal(sim, ref_m[b][1]), b
            Co, Fo = partition.bucket_similarity(Po, nko, np.flatnonzero(g["bucket_of"] == b))
            assert np.array_equal(num, Co) and np.array_equal(sim, Fo), b
            seen.add(b)
    assert seen == set(ref_m)
