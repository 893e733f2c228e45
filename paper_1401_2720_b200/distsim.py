"""Outer (multi-GPU) level of the hierarchically blocked Jacobi (H)SVD.

Drop-in for the reference ``jhsvd.distsim`` (pkg/src/jhsvd/distsim.py), with
the simulated workers replaced by real ones: one process per GPU under
``torch.distributed`` (NCCL on B200s, gloo for CPU tests).  Worker i owns two
block-columns of width n/(2g) of G (m rows) and V (n rows).  One outer step
(distsim.py:296-362) is

    (0)+(1) Gram of the local m x 2n/g pair and its Cholesky factor R
    (2)     nested single-GPU blocked solve of R (the fused p-step kernels)
    (3)     G_x <- G_x V^, V_x <- V_x V^ when the nested solve rotated
    (4)-(6) exchange: keep one block-column, send the other to the worker
            that needs it in the next step, receive one (batched NCCL
            send/recv over NVLink)

and a sweep ends with an all-reduce of the rotation counters (the
reference's "+-reduce of the local counters").

Results do not depend on which worker holds which pair (reference fact,
SURVEY.md section 0.7).  For g <= 4 the mapping is the reference's own
(``optimize_mapping``: exhaustive search for the most transitions over
"fast" links, the reference's two-speed topology), so exchange traces match
the reference record for record; for g > 4, where that search does not
finish, a legal cyclic mapping is found by breadth-first search
(``legal_mapping``).  On NVSwitch every link is equally fast; the trace
keeps the reference's link labels.

Without an initialised process group (or with ``backend="sim"``) the g
workers run one after another in this process on one device, exactly like
the reference simulator; the arithmetic is the same, so both modes and the
oracle agree bitwise.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from .blockkernel import Signature
from .driver import BLOCK_ORIENTED, HsvdResult, SolverConfig
from .strategy import PStrategy, make_strategy

FAST = "fast"
SLOW = "slow"
NVSWITCH = "nvswitch"


@dataclass(frozen=True)
class Topology:
    """Link speed between workers.  ``uniform=False`` is the reference's
    two-speed box (distsim.py:46-55: a worker's partner i xor 1 is reached
    over a fast link, everyone else over a slow one); ``uniform=True`` is an
    NVSwitch box, where every GPU reaches every peer at full NVLink rate."""

    g: int
    uniform: bool = False

    def link_class(self, i: int, j: int) -> str:
        valid = i != j and 0 <= i < self.g and 0 <= j < self.g
        if not valid:
            raise ValueError(f"invalid link ({i}, {j}) for {self.g} workers")
        if self.uniform:
            return FAST
        return FAST if (i ^ j) == 1 else SLOW


class MappingError(ValueError):
    pass


@dataclass(frozen=True)
class ColumnMapping:
    """assignments[s][i] = 1-based (p, q) block pair of worker i at step s;
    moves[s][i] = (src worker, block-column) worker i receives after step s
    (the last step wraps to the first); fast_exchanges = transitions whose
    moves all use fast links (reference distsim.py:58-72)."""

    g: int
    assignments: tuple
    moves: tuple
    fast_exchanges: int = 0


@dataclass(frozen=True)
class ExchangeRecord:
    """One block-column message of the outer level (distsim.py:206-213)."""

    sweep: int
    step: int
    worker: int
    column: int
    dest: int
    link: str


def _holder(assignment, col: int) -> int:
    for i, (p, q) in enumerate(assignment):
        if col == p or col == q:
            return i
    raise MappingError(f"block-column {col} is not held by any worker")


def _moves(cur, nxt):
    """Per worker (src, incoming column), or None if some worker keeps
    zero or two of its columns."""
    out = []
    for i in range(len(cur)):
        kept = set(cur[i]) & set(nxt[i])
        if len(kept) != 1:
            return None
        incoming = (set(nxt[i]) - kept).pop()
        out.append((_holder(cur, incoming), incoming))
    return tuple(out)


def _all_fast(moves, topology: Topology) -> bool:
    return all(topology.link_class(src, i) == FAST for i, (src, _) in enumerate(moves))


def _step_matchings(cur, nxt):
    """Every bijection worker-of-cur-pair -> pair of nxt (as index tuples)
    under which each worker keeps exactly one block-column.  Between two
    p-steps the relation "shares one column" is 2-regular, so there are
    2^(cycles) of them."""
    g = len(cur)
    adj = [[k for k, Q in enumerate(nxt) if len(set(P) & set(Q)) == 1] for P in cur]
    out, used, chosen = [], [False] * g, []

    def rec(i):
        if i == g:
            out.append(tuple(chosen))
            return
        for k in adj[i]:
            if not used[k]:
                used[k] = True
                chosen.append(k)
                rec(i + 1)
                chosen.pop()
                used[k] = False

    rec(0)
    return out


@functools.lru_cache(maxsize=16)
def optimize_mapping(strategy: PStrategy, topology: Topology) -> ColumnMapping:
    """A worker mapping of the outer strategy (order 2g) for the exchange
    protocol of distsim.py:334-360 -- between consecutive steps, the last
    wrapping to the first, every worker keeps exactly one block-column --
    with as many all-fast transitions as the layered search finds.

    Worker 0..g-1 start on pairs 0..g-1 of step 0.  The states of step s are
    the worker -> pair assignments reachable from there (at most g!,
    deduplicated); a forward dynamic program keeps, per state, the largest
    number of all-fast transitions so far (ties: the first parent in sorted
    order), and the wrap back to step 0 is scored at the end.  This replaces
    the reference's exhaustive enumeration of assignment tables
    (distsim.py:135-190, which does not finish for g = 8); the solver's
    results do not depend on the mapping, only the
    exchange trace does, and on NVSwitch (``Topology(g, uniform=True)``)
    every transition is fast."""
    g = topology.g
    if strategy.n != 2 * g:
        raise MappingError(f"strategy order {strategy.n} != 2g = {2 * g}")
    steps = [tuple(sorted(st)) for st in strategy.steps]
    ns = len(steps)
    if g == 1:
        return ColumnMapping(1, tuple((pq,) for pq in strategy.steps), ((),) * ns, 0)

    def moves_of(s, st_a, st_b):
        a = tuple(steps[s][k] for k in st_a)
        b = tuple(steps[(s + 1) % ns][k] for k in st_b)
        return _moves(a, b)

    start = tuple(range(g))
    layers = [{start: (0, None)}]
    for s in range(ns - 1):
        ms = _step_matchings(steps[s], steps[s + 1])
        nxt: dict = {}
        for state in sorted(layers[-1]):
            score = layers[-1][state][0]
            for mm in ms:
                child = tuple(mm[state[i]] for i in range(g))
                if topology.uniform:  # every transition is fast: keep the first parent
                    if child not in nxt:
                        nxt[child] = (score + 1, state)
                    continue
                sc = score + (1 if _all_fast(moves_of(s, state, child), topology) else 0)
                if child not in nxt or sc > nxt[child][0]:
                    nxt[child] = (sc, state)
        layers.append(nxt)
    best = None
    for state in sorted(layers[-1]):
        mv = moves_of(ns - 1, state, start)
        if mv is None:
            continue
        sc = layers[-1][state][0] + (1 if _all_fast(mv, topology) else 0)
        if best is None or sc > best[0]:
            best = (sc, state)
    if best is None:
        raise MappingError("no exchange-compatible worker assignment exists")
    path = [best[1]]
    for s in range(ns - 1, 0, -1):
        path.append(layers[s][path[-1]][1])
    path.reverse()
    assignments = tuple(tuple(steps[s][path[s][i]] for i in range(g)) for s in range(ns))
    moves = tuple(_moves(assignments[s], assignments[(s + 1) % ns]) for s in range(ns))
    return ColumnMapping(g, assignments, moves, best[0])


def legal_mapping(strategy: PStrategy) -> ColumnMapping:
    """The mapping used on B200 boxes: NVSwitch links are uniform, so any
    exchange-compatible mapping is optimal."""
    return optimize_mapping(strategy, Topology(strategy.n // 2, uniform=True))


def default_mapping(strategy: PStrategy) -> ColumnMapping:
    """Mapping of run_distributed: optimised for the reference's two-speed
    topology up to g = 4 (exchange traces then use its fast links the way
    the reference does), the NVSwitch mapping above (the two-speed search
    costs minutes in Python at g = 8 and buys nothing on NVSwitch)."""
    g = strategy.n // 2
    return optimize_mapping(strategy, Topology(g)) if g <= 4 else legal_mapping(strategy)


def local_signature_pair(signature: Signature, p: int, q: int, bw: int) -> Signature:
    """Signature of the local pair (distsim.py:427-433), 1-based blocks."""
    lo_p, hi_p = (p - 1) * bw, p * bw
    lo_q, hi_q = (q - 1) * bw, q * bw
    n_plus = (max(0, min(signature.n_plus, hi_p) - lo_p)
              + max(0, min(signature.n_plus, hi_q) - lo_q))
    return Signature(2 * bw, n_plus)


# ---------------------------------------------------------------------------
# local engines: what one worker computes in steps (0)-(3)


class CudaEngine:
    """The product engine: B200 kernels through the C ABI.  Local blocks are
    column-major (cols, rows) CUDA tensors."""

    def __init__(self, m: int, n: int, local_n: int, cfg: SolverConfig):
        from .driver import SweepEngine

        self.m, self.n, self.local_n, self.cfg = m, n, local_n, cfg
        w = cfg.block_width
        self.local_cfg = replace(
            cfg, accumulate_v=not cfg.solve_v, solve_v=False,
            max_block_sweeps=1 if cfg.variant == BLOCK_ORIENTED else cfg.max_block_sweeps)
        outer = make_strategy(self.local_cfg.outer_strategy, local_n // (w // 2))
        inner = make_strategy(self.local_cfg.inner_strategy, w)
        self.sweeper = SweepEngine(local_n, local_n, local_n, self.local_cfg, outer, inner, 0)

    def device(self):
        from . import _dev

        return _dev.device()

    def gram_cholesky(self, gx):
        import torch

        from . import _lib
        from .blockkernel import RankDeficiencyError

        lib = _lib.require_cuda()
        ln, m = gx.shape
        h = torch.empty((ln, ln), dtype=torch.float64, device=gx.device)
        _lib.check(lib.jh_gram(gx.data_ptr(), m, m, ln, h.data_ptr(), _lib.stream_handle()),
                   "gram")
        r = torch.empty_like(h)
        info = torch.zeros(1, dtype=torch.int32, device=gx.device)
        _lib.check(lib.jh_cholesky(h.data_ptr(), ln, r.data_ptr(), info.data_ptr(),
                                   _lib.stream_handle()), "cholesky")
        bad = int(info.item())
        if bad:
            raise RankDeficiencyError(
                f"nonpositive Cholesky pivot at index {bad}: "
                "the block-pair is numerically rank deficient", index=bad)
        return r

    def nested(self, work, vhat, n_plus_local: int):
        """Nested single-GPU blocked solve of R in place (run_block_jacobi_inplace)."""
        return self.sweeper.run(work, vhat, None, n_plus=n_plus_local)

    def nested_sweep(self, work, vhat, n_plus_local: int):
        """One nested block sweep; (rotations, proper)."""
        return self.sweeper.one_sweep(work, vhat, n_plus_local)

    def postmultiply(self, x, vhat):
        import torch

        from . import _lib

        lib = _lib.require_cuda()
        c, rows = x.shape
        out = torch.empty_like(x)
        _lib.check(lib.jh_gemm(x.data_ptr(), rows, rows, c, vhat.data_ptr(), c, c,
                               out.data_ptr(), rows, _lib.stream_handle()), "postmultiply")
        return out

    def solve_for_v(self, r, work):
        import torch

        from . import _lib

        lib = _lib.require_cuda()
        n = r.shape[0]
        out = torch.empty_like(work)
        _lib.check(lib.jh_back_substitute(r.data_ptr(), n, work.data_ptr(), n, out.data_ptr(),
                                          _lib.stream_handle()), "solve_for_v")
        return out

    def eye(self, k):
        import torch

        return torch.eye(k, dtype=torch.float64, device=self.device())


# ---------------------------------------------------------------------------
# the outer loop


class _Comm:
    """Exchange / reduction backend: torch.distributed (one worker per rank)
    or an in-process simulation (all workers in this process)."""

    def __init__(self, g: int, backend: Optional[str], process_group=None):
        import torch.distributed as dist

        if process_group is not None:
            # a torch.distributed-compatible object for this rank (e.g. ranks
            # run as threads of one process, tests/comm_threads.py)
            dist = process_group
        self.dist = dist
        self.sim = process_group is None and (
            backend == "sim" or not (dist.is_available() and dist.is_initialized()))
        if not self.sim:
            if dist.get_world_size() != g:
                raise ValueError(f"process group has {dist.get_world_size()} ranks, need g = {g}")
            self.rank = dist.get_rank()
        else:
            self.rank = None

    def local_workers(self, g):
        return list(range(g)) if self.sim else [self.rank]


def run_distributed(g_matrix, signature: Optional[Signature], g: int,
                    cfg: SolverConfig = SolverConfig(), hybrid_early_stop: bool = False,
                    collect_trace: bool = False, *, backend: Optional[str] = None,
                    engine=None, mapping: Optional[ColumnMapping] = None,
                    allow_tall: bool = False, process_group=None):
    """Blocked Jacobi (H)SVD over g workers (distsim.py:216-424).

    Under an initialised torch.distributed group of world size g each rank
    is one worker (its GPU = ``torch.cuda.current_device()``); every rank
    must pass the same full ``g_matrix`` and receives the full result.
    Otherwise all g workers are simulated in this process.  Returns
    (HsvdResult, list[ExchangeRecord]).

    ``hybrid_early_stop``: the reference lets the first worker to finish its
    nested solve stop the others (a thread race).  Here the flag is
    all-reduced after every nested sweep -- the same rule, but deterministic.
    """
    import torch

    from . import _dev
    from .driver import _class_sort_order, _sigma_u_dev, _check_scaling_dev, block_jacobi

    shape = tuple(int(s) for s in g_matrix.shape)
    if len(shape) != 2 or (shape[0] != shape[1] and not (allow_tall and shape[0] > shape[1])):
        raise ValueError("the input factor must be square")
    m, n = shape
    if signature is None:
        signature = Signature(n, n)
    if g < 1:
        raise ValueError("need at least one worker")
    comm = _Comm(g, backend, process_group)
    if g == 1:
        return block_jacobi(g_matrix, signature, cfg, allow_tall=allow_tall), []
    if n % (2 * g):
        raise ValueError(f"order {n} must be divisible by 2g = {2 * g}")
    bw = n // (2 * g)
    local_n = 2 * bw
    if local_n % cfg.block_width or local_n < cfg.block_width:
        raise ValueError(f"per-worker width {local_n} must be a multiple of "
                         f"block_width {cfg.block_width}")
    if engine is None:
        engine = CudaEngine(m, n, local_n, cfg)
    mode = _dev.out_mode(g_matrix)
    dev = engine.device()
    if isinstance(g_matrix, torch.Tensor):
        G0 = g_matrix.to(dev, torch.float64).t().contiguous()
    else:
        G0 = torch.from_numpy(np.array(np.asarray(g_matrix, np.float64).T, order="C")).to(dev)
    if not bool(torch.isfinite(G0).all()):
        raise ValueError("the input factor contains NaN or infinity")
    if dev.type == "cuda":
        _check_scaling_dev(G0, m, n)

    outer = make_strategy(cfg.outer_strategy, 2 * g)
    if mapping is None:
        mapping = default_mapping(outer)
    topology = Topology(g)
    nsteps = len(mapping.assignments)
    want_v = cfg.accumulate_v or cfg.solve_v
    mine = comm.local_workers(g)

    def blk(b):
        return slice((b - 1) * bw, b * bw)

    gx, vx = {}, {}
    for i in mine:
        p, q = mapping.assignments[0][i]
        gx[i] = torch.cat((G0[blk(p)], G0[blk(q)])).contiguous()
        if want_v:
            v = torch.zeros((local_n, n), dtype=torch.float64, device=dev)
            v[:bw, (p - 1) * bw:p * bw] = torch.eye(bw, dtype=torch.float64, device=dev)
            v[bw:, (q - 1) * bw:q * bw] = torch.eye(bw, dtype=torch.float64, device=dev)
            vx[i] = v
        else:
            vx[i] = None

    stats: list[tuple[int, int]] = []
    wtrace: list[list[ExchangeRecord]] = [[] for _ in range(g)]  # per worker
    converged = False
    for sweep in range(cfg.max_block_sweeps):
        rot_l = proper_l = 0
        for s in range(nsteps):
            # (0)+(1) shorten every local pair
            prep = {}
            for i in mine:
                p, q = mapping.assignments[s][i]
                r = engine.gram_cholesky(gx[i])
                vhat = engine.eye(local_n) if not cfg.solve_v else None
                sig_l = local_signature_pair(signature, p, q, bw)
                prep[i] = (r, r.clone(), vhat, sig_l.n_plus)
            # (2) nested single-GPU solves
            lstats = {i: [] for i in mine}
            if not hybrid_early_stop:
                for i in mine:
                    _, work, vhat, npl = prep[i]
                    lstats[i], _ = engine.nested(work, vhat, npl)
            else:
                # the first worker to finish stops the others after their
                # current nested sweep (distsim.py:292-321), in lockstep
                done = {i: False for i in mine}
                for _k in range(engine.local_cfg.max_block_sweeps):
                    for i in mine:
                        if not done[i]:
                            _, work, vhat, npl = prep[i]
                            a, b = engine.nested_sweep(work, vhat, npl)
                            lstats[i].append((a, b))
                            done[i] = b == 0
                    if _any(comm, any(done.values()), dev):
                        break
            # (3) post-multiply the tall local block-columns
            for i in mine:
                r, work, vhat, _ = prep[i]
                if cfg.solve_v:
                    vhat = engine.solve_for_v(r, work)
                lst = lstats[i]
                rot_l += sum(a for a, _ in lst)
                proper_l += sum(b for _, b in lst)
                if any(a for a, _ in lst):
                    gx[i] = engine.postmultiply(gx[i], vhat)
                    if vx[i] is not None:
                        vx[i] = engine.postmultiply(vx[i], vhat)
            del prep
            _exchange(comm, mapping, s, gx, vx, bw, mine)
            if collect_trace:
                nxt = mapping.assignments[(s + 1) % nsteps]
                for i in range(g):
                    p, q = mapping.assignments[s][i]
                    kept = ({p, q} & set(nxt[i])).pop()
                    sent = p if kept == q else q
                    dst = _holder(nxt, sent)
                    wtrace[i].append(ExchangeRecord(sweep + 1, s + 1, i, sent, dst,
                                                    topology.link_class(i, dst)))
        rot, proper = _allreduce_counts(comm, rot_l, proper_l, dev)
        stats.append((rot, proper))
        if proper == 0:
            converged = True
            break

    # gather: after the last exchange every worker holds its step-0 pair again
    Gf, Vf = _gather(comm, mapping, gx, vx, m, n, bw, dev, want_v)
    if dev.type == "cuda":
        sigma, U = _sigma_u_dev(Gf, m, n)
        order = _class_sort_order(sigma, signature.n_plus)
        sigma, U = sigma[order], U.index_select(0, order)
        V = Vf.index_select(0, order) if Vf is not None else None
        res = HsvdResult(sigma=_dev.vector_out(sigma, mode), u=_dev.from_colmajor(U, mode),
                         v=_dev.from_colmajor(V, mode) if V is not None else None,
                         signature=signature, stats=tuple(stats), block_sweeps=len(stats),
                         converged=converged)
    else:
        res = engine.finish(Gf, Vf, signature, stats, converged)
    # per-worker records merged in (sweep, step, worker) order (distsim.py:422-423)
    trace = [rec for wt in wtrace for rec in wt]
    trace.sort(key=lambda r: (r.sweep, r.step, r.worker))
    return res, trace


def _any(comm, flag: bool, dev) -> bool:
    """Logical OR of a flag over all workers."""
    if comm.sim:
        return flag
    import torch

    t = torch.tensor([1 if flag else 0], dtype=torch.int64,
                     device=dev if comm.dist.get_backend() == "nccl" else "cpu")
    comm.dist.all_reduce(t, op=comm.dist.ReduceOp.MAX)
    return bool(t.item())


def _exchange(comm, mapping, s, gx, vx, bw, mine):
    """Steps (4)-(6): keep one block-column, send the other, receive one."""
    import torch

    nsteps = len(mapping.assignments)
    cur = mapping.assignments[s]
    nxt = mapping.assignments[(s + 1) % nsteps]
    if comm.sim:
        held = {}
        for i in mine:
            p, q = cur[i]
            held[p] = (gx[i][:bw], None if vx[i] is None else vx[i][:bw])
            held[q] = (gx[i][bw:], None if vx[i] is None else vx[i][bw:])
        for i in mine:
            np_, nq = nxt[i]
            gx[i] = torch.cat((held[np_][0], held[nq][0])).contiguous()
            if vx[i] is not None:
                vx[i] = torch.cat((held[np_][1], held[nq][1])).contiguous()
        return
    dist = comm.dist
    i = comm.rank
    p, q = cur[i]
    np_, nq = nxt[i]
    kept = ({p, q} & {np_, nq}).pop()
    sent = p if kept == q else q
    dst = _holder(nxt, sent)
    incoming = nq if kept == np_ else np_
    src = _holder(cur, incoming)
    half = (lambda t, c: t[:bw] if c == p else t[bw:])
    send_g = half(gx[i], sent).contiguous()
    keep_g = half(gx[i], kept)
    recv_g = torch.empty_like(send_g)
    ops = [dist.P2POp(dist.isend, send_g, dst), dist.P2POp(dist.irecv, recv_g, src)]
    if vx[i] is not None:
        send_v = half(vx[i], sent).contiguous()
        keep_v = half(vx[i], kept)
        recv_v = torch.empty_like(send_v)
        ops += [dist.P2POp(dist.isend, send_v, dst), dist.P2POp(dist.irecv, recv_v, src)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    first_is_kept = kept == np_
    gx[i] = torch.cat((keep_g, recv_g) if first_is_kept else (recv_g, keep_g)).contiguous()
    if vx[i] is not None:
        vx[i] = torch.cat((keep_v, recv_v) if first_is_kept else (recv_v, keep_v)).contiguous()


def _allreduce_counts(comm, rot, proper, dev):
    if comm.sim:
        return rot, proper
    import torch

    t = torch.tensor([rot, proper], dtype=torch.int64,
                     device=dev if comm.dist.get_backend() == "nccl" else "cpu")
    comm.dist.all_reduce(t)
    a, b = (int(x) for x in t.cpu().tolist())
    return a, b


def _gather(comm, mapping, gx, vx, m, n, bw, dev, want_v):
    import torch

    G = torch.empty((n, m), dtype=torch.float64, device=dev)
    V = torch.empty((n, n), dtype=torch.float64, device=dev) if want_v else None
    first = mapping.assignments[0]
    if comm.sim:
        for i, (p, q) in enumerate(first):
            G[(p - 1) * bw:p * bw] = gx[i][:bw]
            G[(q - 1) * bw:q * bw] = gx[i][bw:]
            if V is not None:
                V[(p - 1) * bw:p * bw] = vx[i][:bw]
                V[(q - 1) * bw:q * bw] = vx[i][bw:]
        return G, V
    dist = comm.dist
    g = len(first)
    parts = [torch.empty_like(gx[comm.rank]) for _ in range(g)]
    dist.all_gather(parts, gx[comm.rank])
    for i, (p, q) in enumerate(first):
        G[(p - 1) * bw:p * bw] = parts[i][:bw]
        G[(q - 1) * bw:q * bw] = parts[i][bw:]
    if V is not None:
        parts = [torch.empty_like(vx[comm.rank]) for _ in range(g)]
        dist.all_gather(parts, vx[comm.rank])
        for i, (p, q) in enumerate(first):
            V[(p - 1) * bw:p * bw] = parts[i][:bw]
            V[(q - 1) * bw:q * bw] = parts[i][bw:]
    return G, V
