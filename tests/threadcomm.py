"""In-process stand-in for G ranks on ONE GPU (test infrastructure).

Each rank is a Python thread with its own sa_ctx; the collectives are host
barriers plus device copies, so no kernel ever waits on another kernel (the
ranks' kernels run one after another on the device).  This exercises
sa_partition / sa_redistribute's multi-rank code path -- block ownership,
sample and candidate allgathers, the count exchange, the variable all-to-all
and the receive-side reordering -- and lets the tests check that results do
not depend on the number of ranks (G-invariance)."""
import threading

import numpy as np
import torch

from paper_0905_1744_b200 import binding as B


class ThreadGroup:
    def __init__(self, n):
        self.n = n
        self.barrier = threading.Barrier(n, timeout=120)
        self.slots = [None] * n


class ThreadComm:
    def __init__(self, group: ThreadGroup, rank: int):
        self.g = group
        self.nranks = group.n
        self.rank = rank
        self.errors = []

    def _copy(self, dst, src, nbytes):
        if nbytes:
            B.raw_tensor(dst, nbytes, "cuda").copy_(B.raw_tensor(src, nbytes, "cuda"))

    def allgather(self, user, send, recv, nbytes, stream):
        try:
            torch.cuda.synchronize()
            self.g.slots[self.rank] = (send, nbytes)
            self.g.barrier.wait()
            for r in range(self.nranks):
                src, nb = self.g.slots[r]
                assert nb == nbytes
                self._copy(recv + r * nbytes, src, nbytes)
            torch.cuda.synchronize()
            self.g.barrier.wait()
            return 0
        except Exception as e:  # pragma: no cover
            self.errors.append(repr(e))
            return 1

    def alltoallv(self, user, send, sb, sd, recv, rb, rd, stream):
        try:
            n = self.nranks
            torch.cuda.synchronize()
            self.g.slots[self.rank] = (send, [int(sb[i]) for i in range(n)], [int(sd[i]) for i in range(n)])
            self.g.barrier.wait()
            for r in range(n):
                src, ssb, ssd = self.g.slots[r]
                assert ssb[self.rank] == int(rb[r]), "send/recv sizes disagree"
                self._copy(recv + int(rd[r]), src + ssd[self.rank], ssb[self.rank])
            torch.cuda.synchronize()
            self.g.barrier.wait()
            return 0
        except Exception as e:  # pragma: no cover
            self.errors.append(repr(e))
            return 1

    def ops(self):
        self._ag = B.ALLGATHER_FN(self.allgather)
        self._a2a = B.ALLTOALLV_FN(self.alltoallv)
        return B.sa_comm_ops(None, self._ag, self._a2a)


def run_ranks(G, fn):
    """Run fn(rank, ctx) on G threads with a ThreadComm each; returns results."""
    grp = ThreadGroup(G)
    out = [None] * G
    errs = []

    def body(r):
        try:
            ctx = B.Context()
            if G > 1:
                ctx.attach_comm(ThreadComm(grp, r))
            out[r] = fn(r, ctx)
        except BaseException as e:  # pragma: no cover
            errs.append((r, e))
            grp.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0][1]
    return out
