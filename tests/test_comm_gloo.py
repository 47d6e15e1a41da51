"""The N>1 exchange plumbing on CPU (-m "not gpu"): world_size-2 gloo process
group, the same TorchComm sa_comm_ops callbacks libsa calls on the GPU path,
invoked through their C function pointers with host buffers.  Checks the
allgather rank order and the variable all-to-all's splits / displacements --
the two collectives sa_partition (C1-C3) and sa_redistribute (C4) use."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_0905_1744_b200.binding import TorchComm
        comm = TorchComm(device="cpu")
        ops = comm.ops()
        # allgather: 5 bytes per rank
        send = np.arange(5, dtype=np.uint8) + 10 * rank
        recv = np.zeros(5 * world, dtype=np.uint8)
        rc = ops.allgather(None, send.ctypes.data, recv.ctypes.data, 5, None)
        ok_ag = rc == 0 and recv.tolist() == [i + 10 * r for r in range(world) for i in range(5)]
        # alltoallv: rank r sends (r + d + 1) bytes of value 16*r + d to rank d
        sb = np.array([rank + d + 1 for d in range(world)], dtype=np.int64)
        sd = np.concatenate([[0], np.cumsum(sb)[:-1]]).astype(np.int64)
        rb = np.array([s + rank + 1 for s in range(world)], dtype=np.int64)
        rd = np.concatenate([[0], np.cumsum(rb)[:-1]]).astype(np.int64)
        sbuf = np.concatenate([np.full(sb[d], 16 * rank + d, dtype=np.uint8) for d in range(world)])
        rbuf = np.zeros(int(rb.sum()), dtype=np.uint8)
        P = ctypes.POINTER(ctypes.c_int64)
        rc2 = ops.alltoallv(None, sbuf.ctypes.data, sb.ctypes.data_as(P), sd.ctypes.data_as(P), rbuf.ctypes.data,
                            rb.ctypes.data_as(P), rd.ctypes.data_as(P), None)
        want = np.concatenate([np.full(rb[s], 16 * s + rank, dtype=np.uint8) for s in range(world)])
        ok_a2a = rc2 == 0 and np.array_equal(rbuf, want)
        q.put((rank, ok_ag, ok_a2a, comm.errors))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, False, False, [repr(e)]))


def test_torchcomm_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_ag, ok_a2a, errs in res:
        assert ok_ag and ok_a2a, (rank, errs)
