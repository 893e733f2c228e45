"""Ranks as threads of one process (test infrastructure).

``ThreadWorld(g)`` holds the shared state; ``world.rank(i)`` is a
torch.distributed-compatible object for rank i with the subset the solvers'
non-simulated paths use (get_rank, get_world_size, get_backend, P2POp,
isend, irecv, batch_isend_irecv, all_reduce, all_gather, ReduceOp,
is_available, is_initialized).  Tensors keep their device, so on a one-GPU
box g ranks on cuda:0 drive exactly the code path an NCCL job runs --
send/receive staging, slot bookkeeping, reductions, the final gather --
with CUDA tensors (NCCL itself refuses two ranks on one GPU).

Every rank thread issues its work on the legacy default stream of the
device, so a copy made by one rank is ordered after the kernels that
produced the tensor, whoever launched them.
"""

from __future__ import annotations

import threading
from collections import defaultdict
from enum import Enum


class _ReduceOp(Enum):
    SUM = "sum"
    MIN = "min"
    MAX = "max"


class _Req:
    def __init__(self, fn):
        self._fn = fn

    def wait(self):
        if self._fn is not None:
            self._fn()
            self._fn = None
        return True


class ThreadWorld:
    def __init__(self, g: int, backend: str = "nccl", timeout: float = 600.0):
        self.g = g
        self.backend = backend
        self.timeout = timeout
        self._cv = threading.Condition()
        self._box = defaultdict(list)  # (src, dst) -> FIFO of tensors
        self._coll = {}                 # (kind, seq) -> per-rank contributions
        self._seq = [0] * g
        self._barrier = threading.Barrier(g, timeout=timeout)

    def rank(self, i: int) -> "ThreadRank":
        return ThreadRank(self, i)

    # point to point: a send deposits a copy, a receive takes the oldest
    def _post(self, src, dst, t):
        with self._cv:
            self._box[(src, dst)].append(t.clone())
            self._cv.notify_all()

    def _take(self, src, dst):
        with self._cv:
            if not self._cv.wait_for(lambda: self._box[(src, dst)], timeout=self.timeout):
                raise TimeoutError(f"rank {dst}: nothing from rank {src}")
            return self._box[(src, dst)].pop(0)

    def _collective(self, i, kind, value):
        """Every rank contributes `value`; returns all contributions in rank
        order once the g ranks have arrived."""
        seq = self._seq[i]
        self._seq[i] += 1
        key = (kind, seq)
        with self._cv:
            slot = self._coll.setdefault(key, [None] * self.g)
            slot[i] = value
            self._cv.notify_all()
            if not self._cv.wait_for(lambda: all(v is not None for v in slot),
                                     timeout=self.timeout):
                raise TimeoutError(f"rank {i}: collective {kind} #{seq} incomplete")
            out = list(slot)
        self._barrier.wait()  # nobody reuses the slot before all have read it
        with self._cv:
            self._coll.pop(key, None)
        return out


class ThreadRank:
    ReduceOp = _ReduceOp

    def __init__(self, world: ThreadWorld, i: int):
        self.world = world
        self.i = i

    # -- group queries
    def is_available(self):
        return True

    def is_initialized(self):
        return True

    def get_rank(self):
        return self.i

    def get_world_size(self):
        return self.world.g

    def get_backend(self):
        return self.world.backend

    # -- point to point
    def isend(self, t, dst):
        self.world._post(self.i, dst, t)
        return _Req(None)

    def irecv(self, t, src):
        return _Req(lambda: t.copy_(self.world._take(src, self.i)))

    class P2POp:
        def __init__(self, op, tensor, peer):
            self.op, self.tensor, self.peer = op, tensor, peer

    def batch_isend_irecv(self, ops):
        # sends first (they never block), then the receives
        reqs = [o.op(o.tensor, o.peer) for o in ops if o.op == self.isend]
        reqs += [o.op(o.tensor, o.peer) for o in ops if o.op == self.irecv]
        return reqs

    # -- collectives
    def all_reduce(self, t, op=_ReduceOp.SUM):
        vals = self.world._collective(self.i, "all_reduce", t.clone())
        acc = vals[0].clone()
        for v in vals[1:]:
            if op == _ReduceOp.SUM:
                acc += v
            elif op == _ReduceOp.MIN:
                acc = acc.minimum(v)
            else:
                acc = acc.maximum(v)
        t.copy_(acc)

    def all_gather(self, parts, t):
        vals = self.world._collective(self.i, "all_gather", t.clone())
        for dst, v in zip(parts, vals):
            dst.copy_(v)

    def barrier(self):
        self.world._collective(self.i, "barrier", True)


def run_ranks(g: int, fn, backend: str = "nccl"):
    """fn(rank_index, process_group) on g threads; returns the results in
    rank order (re-raising the first failure)."""
    world = ThreadWorld(g, backend)
    out = [None] * g
    errs = []

    def body(i):
        try:
            out[i] = fn(i, world.rank(i))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            world._barrier.abort()
            with world._cv:
                world._cv.notify_all()

    ths = [threading.Thread(target=body, args=(i,)) for i in range(g)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    return out
