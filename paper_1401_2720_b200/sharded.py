"""Block-column sharding of the two-level solve over N GPUs, bitwise equal to
the single-GPU ``block_jacobi``.

Why this works ("flat" sharding): the row-closest
tables are built by doubling (reference strategy.py:377-404) and rrow is
their reversal, so for any g that divides the blocking, a table of order b
splits into consecutive *segments*: 2g-1 cross segments, in each of which
every pair joins super-column P to super-column M(P) for one perfect
matching M of the 2g super-columns (b/(2g) block-columns each), and one
segment whose pairs stay inside single super-columns.  A GPU that holds a
matched pair of super-columns -- both its G block-columns (m rows) and its V
block-columns (n rows) -- runs every task of the segment that touches them,
b/(2g) tasks per p-step, with the same kernels and the same per-task
arithmetic as one GPU.  Between segments the matchings change like the
steps of a p-strategy of order 2g: each GPU keeps one super-column and
exchanges the other (``optimize_mapping`` over the matchings, NVSwitch
topology), 2g-1 exchanges per sweep, one NCCL send/recv pair of m x n/(2g)
G values plus n x n/(2g) V values.  Counters are all-reduced once per sweep,
and the stop rule is the reference's.  Since every task sees the same data
in the same order, sigma, U, V and the per-sweep statistics are bitwise
those of ``block_jacobi`` (and of the reference's driver.py:251-313) at any
GPU count -- unlike the reference's three-level ``run_distributed``
(distsim.py), whose nested solves are a different algorithm.

Backends: a torch.distributed process group (NCCL over NVLink on a B200
box, one rank per GPU; gloo for CPU tests), or ``backend="sim"``: all g
workers in this process, one after another (tests, and the per-worker
timing of ``tools/project_scaling.py``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .blockkernel import EPS, JDefinitenessError, RankDeficiencyError, Signature
from .distsim import ColumnMapping, optimize_mapping, Topology
from .driver import HsvdResult, SolverConfig
from .strategy import PStrategy, StrategyError, as_table, make_strategy


class ShardingError(ValueError):
    """The pivot table does not split into super-column segments for g."""


@dataclass(frozen=True)
class Segment:
    first: int          # first p-step of the sweep
    nsteps: int
    config: int         # index of the cross matching in effect (mapping step)
    cross: bool         # False: pairs inside super-columns


@dataclass(frozen=True, eq=False)
class ShardPlan:
    g: int
    b: int              # block-columns
    sb: int             # block-columns per super-column (b / 2g)
    segments: tuple     # of Segment, in sweep order
    mapping: ColumnMapping  # over the cross matchings (order 2g, 1-based super-columns)
    table: np.ndarray   # the global pivot table, int32[b-1][b/2][2], 0-based

    def held(self, config: int, worker: int) -> tuple[int, int]:
        """0-based super-columns worker holds in a configuration."""
        p, q = self.mapping.assignments[config][worker]
        return p - 1, q - 1


def _step_matching(pairs: np.ndarray, sb: int, nsc: int):
    """None (pairs inside super-columns), a tuple matching, or False."""
    sp = pairs // sb
    if np.all(sp[:, 0] == sp[:, 1]):
        return None
    mate = {}
    for a, c in sp.tolist():
        if a == c:
            return False
        if mate.setdefault(a, c) != c or mate.setdefault(c, a) != a:
            return False
    if len(mate) != nsc:
        return False
    return tuple(sorted((a + 1, c + 1) for a, c in mate.items() if a < c))


def shard_plan(outer: PStrategy, g: int) -> ShardPlan:
    """Split the outer table into super-column segments for g workers."""
    b = outer.n
    if g < 1 or b % (2 * g):
        raise ShardingError(f"{b} block-columns do not split into {2 * g} super-columns")
    sb = b // (2 * g)
    table = np.asarray(as_table(outer))
    if g == 1:
        one = ColumnMapping(1, (((1, 2),),), ((),), 0)
        return ShardPlan(1, b, sb, (Segment(0, table.shape[0], 0, True),), one, table)
    runs: list[list] = []  # [matching, first, count]
    for s in range(table.shape[0]):
        mt = _step_matching(table[s], sb, 2 * g)
        if mt is False:
            raise ShardingError(f"p-step {s + 1} of the {outer.kind} table mixes super-columns")
        if runs and runs[-1][0] == mt:
            runs[-1][2] += 1
        else:
            runs.append([mt, s, 1])
    cross = [r[0] for r in runs if r[0] is not None]
    if len(cross) != 2 * g - 1 or len(set(cross)) != len(cross):
        raise ShardingError(f"the {outer.kind} table has {len(cross)} cross segments, "
                            f"need {2 * g - 1} distinct matchings")
    try:
        mstrat = PStrategy(2 * g, tuple(cross))
        mapping = optimize_mapping(mstrat, Topology(g, uniform=True))
    except (StrategyError, ValueError) as exc:
        raise ShardingError(f"cross matchings do not form an exchange sequence: {exc}") from exc
    segs = []
    k = -1
    for mt, first, count in runs:
        if mt is not None:
            k += 1
        # a segment inside super-columns runs in the configuration before it
        # (or the first one, when the table starts with it)
        segs.append(Segment(first, count, max(k, 0) if mt is None else k, mt is not None))
    return ShardPlan(g, b, sb, tuple(segs), mapping, table)


@dataclass
class _Local:
    """One worker's block-columns: 2 super-columns in slots 0 / 1."""

    G: object           # (2 sb bw, m) column-major storage
    V: object           # (2 sb bw, n) or None
    slots: list         # 0-based super-column in slot 0, 1


def _local_table(plan: ShardPlan, seg: Segment, slots) -> tuple[np.ndarray, np.ndarray]:
    """Local pivot table of a segment (pairs remapped to slot-local blocks,
    reference order kept) and, per local task, its global task index."""
    sb = plan.sb
    table = plan.table[seg.first:seg.first + seg.nsteps]
    where = {sc: k for k, sc in enumerate(slots)}
    loc = np.empty((seg.nsteps, sb, 2), dtype=np.int32)
    gidx = np.empty((seg.nsteps, sb), dtype=np.int64)
    for s in range(seg.nsteps):
        sp = table[s] // sb
        mine = [t for t in range(table.shape[1]) if sp[t, 0] in where and sp[t, 1] in where]
        if len(mine) != sb:
            raise ShardingError("segment does not give every worker b/(2g) tasks")
        for k, t in enumerate(mine):
            p, q = table[s, t]
            loc[s, k] = (where[p // sb] * sb + p % sb, where[q // sb] * sb + q % sb)
            gidx[s, k] = t
    return loc, gidx


def _gblock(plan: ShardPlan, slots) -> np.ndarray:
    sb = plan.sb
    return np.array([slots[k // sb] * sb + k % sb for k in range(2 * sb)], dtype=np.int32)


# ---------------------------------------------------------------------------
# local engines


class CudaShardEngine:
    """A worker's kernels: the single-GPU sweep kernels (jh_block_sweep) on
    the local pivot table of each segment."""

    def __init__(self, m: int, n: int, plan: ShardPlan, cfg: SolverConfig, n_plus: int,
                 with_v: bool):
        import torch

        from . import _dev, _lib
        from .driver import SweepEngine

        self.lib = _lib.require_cuda()
        self.torch = torch
        self.m, self.n, self.cfg, self.n_plus = m, n, cfg, n_plus
        self.w = cfg.block_width
        self.n_loc = 2 * plan.sb * (self.w // 2)
        self.nv = n if with_v else 0
        self.inner = make_strategy(cfg.inner_strategy, self.w)
        self.dev = _dev.device()
        self._engines: dict = {}
        self.tasks_rotated: list[int] = []          # per sweep, this worker's tasks
        self.tasks_rotated_sweeps: list[int] = []   # per sweep, all workers

    def engine_for(self, key, table, gblock):
        """SweepEngine of one (segment, slot layout) local table (cached)."""
        from .driver import SweepEngine

        eng = self._engines.get(key)
        if eng is None:
            eng = SweepEngine(self.m, self.n_loc, self.nv, self.cfg, None, self.inner,
                              self.n_plus, outer_table=table, gblock=gblock)
            self._engines[key] = eng
        return eng

    def zeros_counters(self):
        c = self.torch.zeros(4, dtype=self.torch.int64, device=self.dev)
        c[2].fill_(-1)
        return c

    def sweep(self, loc: _Local, key, table, gblock, counters):
        eng = self.engine_for(key, table, gblock)
        eng.sweep(loc.G, loc.V, 0, table.shape[0], counters=counters)

    def read(self, counters):
        return [int(x) for x in counters.cpu().tolist()]


# ---------------------------------------------------------------------------
# communication


class _Comm:
    def __init__(self, g: int, backend: Optional[str], process_group=None):
        import torch.distributed as dist

        if process_group is not None:
            # a torch.distributed-compatible object for this rank (e.g. ranks
            # run as threads of one process, tests/comm_threads.py)
            dist = process_group
        self.dist = dist
        self.sim = process_group is None and (
            backend == "sim" or not (dist.is_available() and dist.is_initialized()))
        if not self.sim and dist.get_world_size() != g:
            raise ValueError(f"process group has {dist.get_world_size()} ranks, need g = {g}")
        self.rank = None if self.sim else dist.get_rank()

    def workers(self, g):
        return list(range(g)) if self.sim else [self.rank]

    def all_sum(self, vals, dev):
        if self.sim:
            return vals
        import torch

        t = torch.tensor(vals, dtype=torch.int64,
                         device=dev if self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t)
        return [int(x) for x in t.cpu().tolist()]

    def all_min(self, val: int, dev) -> int:
        if self.sim:
            return val
        import torch

        t = torch.tensor([val], dtype=torch.int64,
                         device=dev if self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return int(t.item())


def _exchange(comm: _Comm, plan: ShardPlan, cfg_from: int, cfg_to: int, locs: dict,
              bwc: int, stage: dict):
    """Move super-columns from the holders of configuration cfg_from to those
    of cfg_to; every worker keeps one slot and refills the other."""
    g = plan.g
    holder = {}
    for i in range(g):
        for sc in plan.held(cfg_from, i):
            holder[sc] = i
    plans = {}
    for i in range(g):
        cur, nxt = set(plan.held(cfg_from, i)), set(plan.held(cfg_to, i))
        keep = cur & nxt
        if len(keep) != 1:
            raise ShardingError("exchange must keep exactly one super-column per worker")
        out_sc = (cur - keep).pop()
        in_sc = (nxt - keep).pop()
        plans[i] = (out_sc, in_sc, holder[in_sc])
    dest = {plans[i][1]: i for i in range(g)}  # super-column -> its next holder
    if comm.sim:
        import torch

        staged = {}
        for i in locs:
            out_sc, _, _ = plans[i]
            k = locs[i].slots.index(out_sc)
            sl = slice(k * bwc, (k + 1) * bwc)
            staged[out_sc] = (locs[i].G[sl].clone(),
                              None if locs[i].V is None else locs[i].V[sl].clone())
        for i in locs:
            out_sc, in_sc, _ = plans[i]
            k = locs[i].slots.index(out_sc)
            sl = slice(k * bwc, (k + 1) * bwc)
            locs[i].G[sl].copy_(staged[in_sc][0])
            if locs[i].V is not None:
                locs[i].V[sl].copy_(staged[in_sc][1])
            locs[i].slots[k] = in_sc
        del staged, torch
        return
    dist = comm.dist
    i = comm.rank
    loc = locs[i]
    out_sc, in_sc, src = plans[i]
    k = loc.slots.index(out_sc)
    sl = slice(k * bwc, (k + 1) * bwc)
    dst = dest[out_sc]
    rg, rv = stage["G"], stage.get("V")
    ops = [dist.P2POp(dist.isend, loc.G[sl], dst), dist.P2POp(dist.irecv, rg, src)]
    if loc.V is not None:
        ops += [dist.P2POp(dist.isend, loc.V[sl], dst), dist.P2POp(dist.irecv, rv, src)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    loc.G[sl].copy_(rg)
    if loc.V is not None:
        loc.V[sl].copy_(rv)
    loc.slots[k] = in_sc


# ---------------------------------------------------------------------------
# driver


def block_jacobi_sharded(g_matrix, signature: Optional[Signature], g: int,
                         cfg: SolverConfig = SolverConfig(), *, backend: Optional[str] = None,
                         engine=None, timer: Optional[Callable] = None,
                         allow_tall: bool = False, process_group=None) -> HsvdResult:
    """``block_jacobi`` with the block-columns sharded over g workers (one
    per rank of the initialised torch.distributed group, or simulated in
    this process); bitwise equal to ``block_jacobi`` for every g.  Every rank
    passes the same full factor and receives the full result.  ``timer``
    (sim mode) is called as timer(worker, segment_index, start|stop).
    ``process_group``: a torch.distributed-compatible object to use instead
    of the global process group (one per rank)."""
    import torch

    from . import _dev
    from .driver import _check_scaling_dev, _class_sort_order, _sigma_u_dev, block_jacobi

    shape = tuple(int(s) for s in g_matrix.shape)
    if len(shape) != 2 or (shape[0] != shape[1] and not (allow_tall and shape[0] > shape[1])):
        raise ValueError("the input factor must be square")
    m, n = shape
    if signature is None:
        signature = Signature(n, n)
    if signature.n != n:
        raise ValueError("signature order does not match the matrix")
    w = cfg.block_width
    if n % w or n < w:
        raise ValueError(f"order {n} must be a positive multiple of block_width {w}")
    if cfg.solve_v or cfg.shortening != "cholesky":
        raise NotImplementedError("the sharded solve supports Cholesky shortening with V "
                                  "accumulated or not (solve_v: use block_jacobi)")
    comm = _Comm(g, backend, process_group)
    if g == 1 and engine is None and comm.sim:
        return block_jacobi(g_matrix, signature, cfg, allow_tall=allow_tall)
    bw = w // 2
    b = n // bw
    outer = make_strategy(cfg.outer_strategy, b)
    plan = shard_plan(outer, g)
    mode = _dev.out_mode(g_matrix)
    with_v = cfg.accumulate_v
    if engine is None:
        engine = CudaShardEngine(m, n, plan, cfg, signature.n_plus, with_v)
    dev = engine.dev
    if isinstance(g_matrix, torch.Tensor):
        G0 = g_matrix.to(dev, torch.float64).t().contiguous()
    else:
        G0 = torch.from_numpy(np.array(np.asarray(g_matrix, np.float64).T, order="C")).to(dev)
    if not bool(torch.isfinite(G0).all()):
        raise ValueError("the input factor contains NaN or infinity")
    if dev.type == "cuda":
        _check_scaling_dev(G0, m, n)
    bwc = plan.sb * bw  # columns per super-column
    mine = comm.workers(g)
    first_cfg = plan.segments[0].config
    locs = {}
    for i in mine:
        slots = list(plan.held(first_cfg, i))
        Gl = torch.cat([G0[sc * bwc:(sc + 1) * bwc] for sc in slots]).contiguous()
        Vl = None
        if with_v:
            Vl = torch.zeros((2 * bwc, n), dtype=torch.float64, device=dev)
            for k, sc in enumerate(slots):
                Vl[k * bwc:(k + 1) * bwc, sc * bwc:(sc + 1) * bwc] = torch.eye(
                    bwc, dtype=torch.float64, device=dev)
        locs[i] = _Local(Gl, Vl, slots)
    del G0
    stage = {}
    if not comm.sim:
        stage["G"] = torch.empty((bwc, m), dtype=torch.float64, device=dev)
        if with_v:
            stage["V"] = torch.empty((bwc, n), dtype=torch.float64, device=dev)
    # local tables per (segment, slot layout), built on first use
    tables: dict = {}

    def table_for(si, seg, slots):
        key = (si, tuple(slots))
        if key not in tables:
            tables[key] = _local_table(plan, seg, slots) + (_gblock(plan, slots),)
        return key, tables[key]

    stats: list[tuple[int, int]] = []
    converged = False
    cur_cfg = first_cfg
    rot_local: list[int] = []
    rot_all: list[int] = []
    for _ in range(cfg.max_block_sweeps):
        per = {i: [] for i in mine}
        for si, seg in enumerate(plan.segments):
            if seg.config != cur_cfg:
                _exchange(comm, plan, cur_cfg, seg.config, locs, bwc, stage)
                cur_cfg = seg.config
            for i in mine:
                key, (tab, gidx, gblk) = table_for(si, seg, locs[i].slots)
                cnt = engine.zeros_counters()
                if timer:
                    timer(i, si, "start")
                engine.sweep(locs[i], key, tab, gblk, cnt)
                if timer:
                    timer(i, si, "stop")
                per[i].append((cnt, seg, gidx))
        rot = proper = nrot = 0
        first_err = (1 << 62)
        for i in mine:
            for cnt, seg, gidx in per[i]:
                r, p, key, nr = engine.read(cnt)
                rot += r
                proper += p
                nrot += nr
                if key != -1:
                    key &= (1 << 64) - 1
                    ps, task = key >> 38, (key >> 16) & 0x3FFFFF
                    status, index = (key >> 13) & 7, key & 0x1FFF
                    gs = seg.first + ps
                    enc = (gs << 40) | (int(gidx[ps, task]) << 16) | (status << 13) | index
                    first_err = min(first_err, enc)
        rot_local.append(nrot)
        rot, proper, nrot = comm.all_sum([rot, proper, nrot], dev)
        rot_all.append(nrot)
        first_err = comm.all_min(first_err, dev)
        if first_err != (1 << 62):
            _raise(first_err, plan, bw)
        stats.append((rot, proper))
        if proper == 0:
            converged = True
            break

    if hasattr(engine, "tasks_rotated"):
        engine.tasks_rotated = rot_local
        engine.tasks_rotated_sweeps = rot_all
    Gf, Vf = _gather(comm, plan, locs, m, n, bwc, dev, with_v)
    if dev.type != "cuda":
        return engine.finish(Gf, Vf, signature, stats, converged)
    sigma, U = _sigma_u_dev(Gf, m, n)
    order = _class_sort_order(sigma, signature.n_plus)
    sigma, U = sigma[order], U.index_select(0, order)
    V = Vf.index_select(0, order) if Vf is not None else None
    return HsvdResult(sigma=_dev.vector_out(sigma, mode), u=_dev.from_colmajor(U, mode),
                      v=_dev.from_colmajor(V, mode) if V is not None else None,
                      signature=signature, stats=tuple(stats), block_sweeps=len(stats),
                      converged=converged)


def _raise(enc: int, plan: ShardPlan, bw: int):
    gs, task = enc >> 40, (enc >> 16) & 0xFFFFFF
    status, index = (enc >> 13) & 7, enc & 0x1FFF
    if status == 1:
        raise RankDeficiencyError(
            f"nonpositive Cholesky pivot at index {index}: "
            "the block-pair is numerically rank deficient", index=index)
    if status == 2:
        p, q = (int(x) for x in plan.table[gs, task])
        gcol = (p * bw + index) if index <= bw else (q * bw + index - bw)
        raise RankDeficiencyError(f"zero column norm at local column {index} (global {gcol})",
                                  index=index)
    raise JDefinitenessError(f"hyperbolic pivot at local column {index} has |coth 2phi| < 1")


def _gather(comm: _Comm, plan: ShardPlan, locs: dict, m: int, n: int, bwc: int, dev,
            with_v: bool):
    import torch

    G = torch.empty((n, m), dtype=torch.float64, device=dev)
    V = torch.empty((n, n), dtype=torch.float64, device=dev) if with_v else None

    def place(slots, gl, vl):
        for k, sc in enumerate(slots):
            G[sc * bwc:(sc + 1) * bwc] = gl[k * bwc:(k + 1) * bwc]
            if V is not None:
                V[sc * bwc:(sc + 1) * bwc] = vl[k * bwc:(k + 1) * bwc]

    if comm.sim:
        for loc in locs.values():
            place(loc.slots, loc.G, loc.V)
        return G, V
    dist = comm.dist
    loc = locs[comm.rank]
    g = plan.g
    gparts = [torch.empty_like(loc.G) for _ in range(g)]
    dist.all_gather(gparts, loc.G)
    vparts = None
    if with_v:
        vparts = [torch.empty_like(loc.V) for _ in range(g)]
        dist.all_gather(vparts, loc.V)
    sl = torch.tensor(loc.slots, dtype=torch.int64,
                      device=dev if dist.get_backend() == "nccl" else "cpu")
    slots_all = [torch.empty_like(sl) for _ in range(g)]
    dist.all_gather(slots_all, sl)
    for r in range(g):
        place([int(x) for x in slots_all[r].cpu().tolist()], gparts[r],
              vparts[r] if vparts is not None else None)
    return G, V
