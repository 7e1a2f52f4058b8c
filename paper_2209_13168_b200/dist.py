"""Multi-GPU: one process per GPU (torch.distributed), sharding where the path
shards naturally.

* ``estimate_stream_divergence_dist`` -- independent windows of a landing
  sequence split into contiguous blocks balanced by event count; every rank
  solves its block on its own GPU (one evd_solve_windows launch); the
  per-window samples (a few scalars each) are all-gathered.  No image
  all-reduce, no data-path collective.
* ``solve_batched`` -- one window's best-first BnB with a batched frontier:
  each round pops up to ``k`` open nodes, evaluates all their centres and
  children in one pass, and keeps the reference's incumbent (>=) and pruning
  (>=) rules.  With a process group the round's evaluations are split over
  the ranks (events replicated on every GPU: S_bar is not additive over event
  shards) and their results all-gathered (one small tensor per round), so
  every rank holds the identical BnB state.  Certified within gamma of the
  global optimum like the reference (SURVEY §8(c) parity P3).
* ``broadcast_window`` / ``solve_batched_dist`` -- the window's events go from
  one rank to every GPU once (one packed float64 tensor, NCCL broadcast over
  NVLink) and are loaded into each rank's libevd context from device memory.

The evaluators are injectable so the host logic runs under ``gloo`` on CPU
(tests/test_dist.py); on GPUs they default to the libevd entry points.
"""

from __future__ import annotations

import heapq
import itertools
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from .geometry import DivergenceSample, divergence_from_velocity, velocity_domain


# ------------------------------------------------------------------ windows
def shard_bounds(sizes: Sequence[int], world: int) -> list[tuple[int, int]]:
    """Contiguous [start, stop) window blocks, one per rank, balanced by
    total events (prefix split at the k/world quantiles)."""
    sizes = np.asarray(sizes, dtype=np.float64) + 1.0  # empty windows still cost a little
    cum = np.concatenate([[0.0], np.cumsum(sizes)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        j = int(np.searchsorted(cum, target, side="left"))
        if j > 0 and (j >= len(cum) or target - cum[j - 1] <= cum[j] - target):
            j -= 1  # the prefix boundary closest to the quantile
        cuts.append(j)
    cuts.append(len(sizes))
    cuts = np.maximum.accumulate(np.clip(cuts, 0, len(sizes)))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def estimate_stream_divergence_dist(batches, params, group=None,
                                    solve_local: Callable | None = None):
    """estimate_stream_divergence (solver.py:139-162) with windows sharded over
    the ranks of ``group`` (torch.distributed); returns the full sample list on
    every rank, in window order."""
    import torch.distributed as dist

    if solve_local is None:
        from .solver import estimate_stream_divergence as solve_local
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = shard_bounds([b.n for b in batches], world)[rank]
    local = solve_local(batches[lo:hi], params)
    if world == 1:
        return local
    gathered = [None] * world
    dist.all_gather_object(gathered, [(s.t, s.divergence, s.contrast, s.bound_gap,
                                       s.iterations, s.runtime) for s in local], group=group)
    out = []
    for part in gathered:
        out.extend(DivergenceSample(*row) for row in part)
    return out


# ------------------------------------------------------------------ batched / split BnB
@dataclass(frozen=True)
class BatchedResult:
    nu: float
    contrast: float
    bound_gap: float
    rounds: int          # dependent evaluation rounds (launch batches)
    nodes: int           # expanded nodes (centre evaluations)
    bound_evals: int     # bound evaluations incl. the root


def gpu_evaluators(batch, ctx=None):
    """(centres -> contrasts, (lo, hi) -> c_bar) on this process's GPU; the
    window is loaded once (or is already resident in ``ctx``)."""
    from .contrast import assemble_bound, frontier_terms, load_window, point_terms

    ctx = ctx if ctx is not None else load_window(batch)
    m = batch.geometry.n_pixels

    def contrasts(nus):
        return point_terms(batch, nus, ctx=ctx, loaded=True)[1]

    def bounds(lo, hi):
        s, fi, _ = frontier_terms(batch, lo, hi, ctx=ctx, loaded=True)
        return np.array([assemble_bound(int(a), int(b), m).c_bar for a, b in zip(s, fi)])

    return contrasts, bounds


def gpu_node_evaluator(batch, ctx=None):
    """nodes (lo[], hi[]) -> (centre contrasts, child c_bar lo, child c_bar
    hi) on this process's GPU, several nodes per event pass (evd_eval_nodes)."""
    from .contrast import load_window, node_terms

    ctx = ctx if ctx is not None else load_window(batch)

    def nodes(lo, hi):
        return node_terms(batch, lo, hi, ctx=ctx, loaded=True)

    return nodes


def _coll_device(group):
    """Tensor device for collectives: the rank's GPU under NCCL, else the CPU."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _split_eval(fn, args, group, per_item: int = 1):
    """Evaluate fn over the items of ``args`` split round-robin over the ranks
    and all-gather the results (identical arrays on every rank): one padded
    float64 tensor per rank, all-gathered over the group's backend.  fn
    returns ``per_item`` values per item, item-major."""
    import torch
    import torch.distributed as dist

    if group is None and not dist.is_initialized():
        return np.asarray(fn(*args), dtype=np.float64)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = len(args[0])
    mine = np.arange(rank, n, world)
    vals = np.asarray(fn(*[np.asarray(a)[mine] for a in args]), dtype=np.float64) if len(mine) else \
        np.empty(0)
    width = -(-n // world) * per_item  # ceil: rank r holds items r, r + world, ...
    dev = _coll_device(group)
    local = torch.zeros(width, dtype=torch.float64, device=dev)
    local[: len(vals)] = torch.from_numpy(vals).to(dev)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    out = np.empty((n, per_item), dtype=np.float64)
    for r, part in enumerate(parts):
        idx = np.arange(r, n, world)
        out[idx] = part[: len(idx) * per_item].cpu().numpy().reshape(-1, per_item)
    return out.ravel() if per_item > 1 else out[:, 0]


def broadcast_window(batch, group=None, src: int = 0):
    """The window's events from rank ``src`` to every rank: one
    packed float64 tensor [x | y | t] broadcast over the group's backend (NCCL:
    GPU to GPU over NVLink).  Ranks other than ``src`` pass ``batch=None``.
    Returns (x, y, t, tau, geometry), tensors on the collective device."""
    import torch
    import torch.distributed as dist

    from .events import SensorGeometry
    dev = _coll_device(group)
    rank = dist.get_rank(group)
    meta = torch.zeros(4, dtype=torch.float64, device=dev)
    if rank == src:
        g = batch.geometry
        meta[:] = torch.tensor([batch.n, g.width, g.height, float(batch.tau)], dtype=torch.float64)
    dist.broadcast(meta, src=src, group=group)
    n, w, h, tau = int(meta[0]), int(meta[1]), int(meta[2]), float(meta[3])
    buf = torch.empty(3 * n, dtype=torch.float64, device=dev)
    if rank == src:
        host = np.concatenate([np.asarray(batch.x, np.float64), np.asarray(batch.y, np.float64),
                               np.asarray(batch.t, np.float64)])
        buf.copy_(torch.from_numpy(host))
    dist.broadcast(buf, src=src, group=group)
    return buf[:n], buf[n:2 * n], buf[2 * n:], tau, SensorGeometry(w, h)


def solve_batched_dist(batch, params, k: int = 64, group=None, src: int = 0) -> "BatchedResult":
    """``solve_batched`` over the ranks of ``group`` on GPUs: events broadcast
    once from ``src`` and loaded from device memory, each round's evaluations
    split over the ranks.  Every rank returns the identical result."""
    from types import SimpleNamespace

    from .contrast import load_window_device
    x, y, t, tau, geometry = broadcast_window(batch, group, src)
    ctx = load_window_device(x, y, t, tau, geometry)
    view = SimpleNamespace(n=int(t.numel()), tau=tau, geometry=geometry)
    contrasts, bounds = gpu_evaluators(view, ctx=ctx)
    return solve_batched(view, params, k=k, contrasts=contrasts, bounds=bounds, group=group,
                         split=True)


def solve_batched(batch, params, k: int = 64, contrasts: Callable | None = None,
                  bounds: Callable | None = None, group=None,
                  split: bool = False) -> BatchedResult:
    """Best-first BnB popping up to ``k`` nodes per round.

    Rules per node are the reference's (solver.py:102-119); the order of
    expansion differs (a round expands the k best open nodes), so the result
    is certified within gamma of the optimum rather than bit-identical.
    ``split``: divide each round's evaluations over the ranks of ``group``.
    """
    if contrasts is None or bounds is None:
        contrasts, bounds = gpu_evaluators(batch)
    ev_c = (lambda nus: _split_eval(contrasts, (nus,), group)) if split else contrasts
    ev_b = (lambda lo, hi: _split_eval(bounds, (lo, hi), group)) if split else bounds
    dom = velocity_domain(batch.tau, params.epsilon)
    nu_hat = dom.center
    c_hat = float(np.asarray(ev_c(np.array([nu_hat])))[0])
    root = float(np.asarray(ev_b(np.array([dom.lo]), np.array([dom.hi])))[0])
    ctr = itertools.count()
    heap = [(-root, next(ctr), dom.lo, dom.hi)]
    rounds = nodes = 0
    evals = 1
    gap_out = 0.0
    while heap:
        # the reference's stop test on the best open node (solver.py:105-108)
        neg, _, lo, hi = heap[0]
        gap = -neg - c_hat
        if gap <= params.gamma or hi - lo < params.min_interval_width:
            gap_out = max(gap, 0.0)
            break
        batch_nodes = []
        # never expand past the cap: the reference raises right after the node
        # that reaches it (solver.py:118-119)
        room = min(k, params.max_iterations - nodes)
        while heap and len(batch_nodes) < room:
            neg, _, lo, hi = heap[0]
            if -neg - c_hat <= params.gamma or hi - lo < params.min_interval_width:
                break
            heapq.heappop(heap)
            batch_nodes.append((lo, hi))
        rounds += 1
        nodes += len(batch_nodes)
        cen = np.array([0.5 * (lo + hi) for lo, hi in batch_nodes])
        cc = np.asarray(ev_c(cen))
        clo = np.array([v for (lo, hi), c in zip(batch_nodes, cen) for v in (lo, c)])
        chi = np.array([v for (lo, hi), c in zip(batch_nodes, cen) for v in (c, hi)])
        cb = np.asarray(ev_b(clo, chi))
        evals += len(clo)
        for c, v in zip(cen, cc):  # incumbent update with >= (solver.py:111)
            if v >= c_hat:
                nu_hat, c_hat = float(c), float(v)
        for lo, hi, b in zip(clo, chi, cb):
            if b >= c_hat:  # solver.py:116
                heapq.heappush(heap, (-float(b), next(ctr), float(lo), float(hi)))
        if nodes >= params.max_iterations:  # solver.py:118-119, incumbent carried
            from .solver import IterationLimitError
            raise IterationLimitError(nu_hat, c_hat, nodes)
    return BatchedResult(nu_hat, c_hat, gap_out, rounds, nodes, evals)


# ------------------------------------------------------------------ exact speculative split BnB
@dataclass(frozen=True)
class SpecResult:
    nu: float
    contrast: float
    bound_gap: float
    iterations: int      # the reference's pops (identical to maximise_contrast_bnb)
    rounds: int          # evaluation rounds (one split evaluation + all-gather each)
    node_evals: int      # nodes evaluated (centre + both children), speculation included
    bound_evals: int     # bound evaluations made (root + children of evaluated nodes)


def solve_spec(batch, params, slots: int = 8, contrasts: Callable | None = None,
               bounds: Callable | None = None, group=None, split: bool = False,
               nodes: Callable | None = None) -> SpecResult:
    """The reference's best-first BnB (solver.py:79-123) replayed exactly,
    with node evaluations batched speculatively -- the host form of
    k_solve_spec's rounds, made to spread over ranks.

    A node's results (centre contrast, both child bounds) are a pure function
    of its interval, so they can be computed before the reference pops it.
    Each round evaluates ``slots`` nodes: the node the replay must pop next
    (the first one not yet evaluated) and the best other open entries that
    could still be popped (bound above c_hat + gamma, width >= the minimum).
    The replay then pops in the reference's order -- heap key (-c_bar,
    push counter), incumbent update with >=, pruning with >=, the iteration
    cap after the node -- for as long as the popped nodes are evaluated.
    ``split``: each round's nodes are divided over the ranks of ``group``
    (events replicated; ``_split_eval``) and their results all-gathered, so
    every rank holds the same cache and replays the same pops.  Results,
    including the pop count, are the reference's on any number of ranks.

    Evaluators: ``nodes(lo[], hi[]) -> (contrast[], cbar_lo[], cbar_hi[])``
    (one call per round, e.g. ``gpu_node_evaluator``), else ``contrasts`` and
    ``bounds`` (two calls per round); ``bounds`` also gives the root's bound.
    """
    from .solver import IterationLimitError

    if bounds is None or (nodes is None and contrasts is None):
        contrasts, bounds = gpu_evaluators(batch)
    if nodes is None:
        def nodes(lo, hi):
            cen = 0.5 * (lo + hi)  # VelocityInterval.center, elementwise
            cb = np.asarray(bounds(np.stack([lo, cen], 1).ravel(), np.stack([cen, hi], 1).ravel()))
            return np.asarray(contrasts(cen)), cb[0::2], cb[1::2]

    def node_rows(lo, hi):  # item-major (contrast, cbar_lo, cbar_hi) per node
        return np.stack([np.asarray(v, np.float64) for v in nodes(lo, hi)], 1).ravel()

    def ev_nodes(lo, hi):
        flat = _split_eval(node_rows, (lo, hi), group, per_item=3) if split else node_rows(lo, hi)
        return np.asarray(flat, np.float64).reshape(-1, 3)

    dom = velocity_domain(batch.tau, params.epsilon)
    cache: dict[tuple[float, float], tuple[float, float, float]] = {}
    rounds = node_evals = 0
    bound_evals = 1

    def evaluate(todo):
        nonlocal rounds, node_evals, bound_evals
        r = ev_nodes(np.array([a for a, _ in todo], dtype=np.float64),
                     np.array([b for _, b in todo], dtype=np.float64))
        for j, node in enumerate(todo):
            cache[node] = (float(r[j, 0]), float(r[j, 1]), float(r[j, 2]))
        rounds += 1
        node_evals += len(todo)
        bound_evals += 2 * len(todo)

    root = (dom.lo, dom.hi)
    # round 0: the root's bound (solver.py:96-98, split like any evaluation)
    # and the root as a node, whose centre contrast is the initial incumbent
    # (solver.py:93-94: the same point)
    ev_b = (lambda lo, hi: _split_eval(bounds, (lo, hi), group)) if split else bounds
    root_bound = float(np.asarray(ev_b(np.array([dom.lo]), np.array([dom.hi])))[0])
    evaluate([root])
    nu_hat, c_hat = dom.center, cache[root][0]
    ctr = itertools.count()
    heap = [(-root_bound, next(ctr), dom.lo, dom.hi)]
    iterations = 0
    bound_gap = 0.0
    while heap:
        neg, _, lo, hi = heap[0]
        gap = -neg - c_hat
        if gap <= params.gamma or hi - lo < params.min_interval_width:  # solver.py:105-108
            iterations += 1
            bound_gap = max(gap, 0.0)
            break
        if (lo, hi) not in cache:
            # next round: this node, then the best open entries the replay may pop
            todo = [(lo, hi)]
            for e in heapq.nsmallest(len(heap), heap):
                if len(todo) >= slots:
                    break
                elo, ehi = e[2], e[3]
                if (elo, ehi) in cache or (elo, ehi) == (lo, hi):
                    continue
                if -e[0] - c_hat <= params.gamma or ehi - elo < params.min_interval_width:
                    continue  # popping it ends the search: never evaluated
                todo.append((elo, ehi))
            evaluate(todo)
        heapq.heappop(heap)
        iterations += 1
        cen = 0.5 * (lo + hi)
        c_c, cb_lo, cb_hi = cache[(lo, hi)]
        if c_c >= c_hat:  # solver.py:111-113
            nu_hat, c_hat = cen, c_c
        for clo, chi, b in ((lo, cen, cb_lo), (cen, hi, cb_hi)):
            if b >= c_hat:  # solver.py:116
                heapq.heappush(heap, (-b, next(ctr), clo, chi))
        if iterations >= params.max_iterations:  # solver.py:118-119
            raise IterationLimitError(nu_hat, c_hat, iterations)
    return SpecResult(nu_hat, c_hat, bound_gap, iterations, rounds, node_evals, bound_evals)


def solve_spec_dist(batch, params, slots_per_rank: int = 4, group=None,
                    src: int = 0) -> SpecResult:
    """``solve_spec`` over the ranks of ``group`` on GPUs: the window's events
    broadcast once from ``src`` (NCCL) and loaded from device memory, each
    round's ``slots_per_rank * world`` node evaluations split over the ranks.
    Every rank returns the identical, reference-exact result."""
    import torch.distributed as dist
    from types import SimpleNamespace

    from .contrast import load_window_device
    x, y, t, tau, geometry = broadcast_window(batch, group, src)
    ctx = load_window_device(x, y, t, tau, geometry)
    view = SimpleNamespace(n=int(t.numel()), tau=tau, geometry=geometry)
    contrasts, bounds = gpu_evaluators(view, ctx=ctx)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    return solve_spec(view, params, slots=slots_per_rank * world, bounds=bounds,
                      nodes=gpu_node_evaluator(view, ctx=ctx), group=group, split=world > 1)


def divergence_of(result, tau: float) -> float:
    return divergence_from_velocity(result.nu, tau)
