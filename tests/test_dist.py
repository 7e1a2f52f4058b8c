"""Multi-process host logic of the multi-GPU paths, world_size 2 over gloo (CPU).

The device evaluators are replaced by the pinned CPU oracle, so these tests
check the sharding, the all-gathers and the replicated batched BnB state.
"""

import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT, f64
from oracle import oracle as orc
from paper_2209_13168_b200 import dist as pdist
from paper_2209_13168_b200.geometry import DivergenceSample, divergence_from_velocity
from paper_2209_13168_b200.solver import IterationLimitError, SolverParams


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_evaluators(batch):
    def contrasts(nus):
        return np.array([orc.contrast_at(batch, float(nu)) for nu in nus])

    def bounds(lo, hi):
        return np.array([orc.bound_terms(batch, float(a), float(b))[2] for a, b in zip(lo, hi)])

    return contrasts, bounds


def _oracle_stream(batches, params):
    out = []
    for b in batches:
        if b.n == 0:
            continue
        r = orc.maximise_contrast_bnb(b)
        out.append(DivergenceSample(b.t_end, divergence_from_velocity(r.nu, b.tau), r.contrast,
                                    r.bound_gap, r.iterations, 0.0))
    return out


def _windows():
    from paper_2209_13168_b200 import synth
    d = synth.Descent(64, 64, 300, nu=-0.4, duration=2.0, seed=11)
    return synth.stream_windows(synth.landing_stream(d), 0.5)


def _worker(rank, world, port, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = SolverParams()
        wins = _windows()
        samples = pdist.estimate_stream_divergence_dist(wins, params, solve_local=_oracle_stream)
        b = wins[1]
        c, bd = _oracle_evaluators(b)
        res = pdist.solve_batched(b, params, k=8, contrasts=c, bounds=bd, split=True)
        # the iteration cap holds in the split solve too, incumbent carried
        try:
            pdist.solve_batched(b, SolverParams(max_iterations=3), k=2, contrasts=c, bounds=bd,
                                split=True)
            capped = None
        except IterationLimitError as e:
            capped = (e.nu, e.contrast, e.iterations)
        # the window's events from rank 0 to every rank (one packed broadcast)
        x, y, t, tau, geom = pdist.broadcast_window(b if rank == 0 else None)
        same = (np.array_equal(x.numpy(), b.x) and np.array_equal(y.numpy(), b.y) and
                np.array_equal(t.numpy(), b.t) and tau == b.tau and geom == b.geometry)
        # the exact speculative solve, each round's evaluations split over the ranks
        sp = pdist.solve_spec(b, params, slots=6, contrasts=c, bounds=bd, split=True)
        try:
            pdist.solve_spec(b, SolverParams(max_iterations=4), slots=4, contrasts=c, bounds=bd,
                             split=True)
            sp_cap = None
        except IterationLimitError as e:
            sp_cap = (e.nu, e.contrast, e.iterations)
        queue.put((rank, [(s.t, s.contrast, s.iterations) for s in samples],
                   (res.nu, res.contrast, res.rounds, res.nodes), same, capped,
                   (sp.nu, sp.contrast, sp.bound_gap, sp.iterations, sp.rounds), sp_cap))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_balanced_and_contiguous():
    sizes = [10, 0, 30, 30, 5, 5, 100, 20]
    for world in (1, 2, 3, 8):
        b = pdist.shard_bounds(sizes, world)
        assert b[0][0] == 0 and b[-1][1] == len(sizes)
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
    two = pdist.shard_bounds(sizes, 2)
    assert two == [(0, 6), (6, 8)]


def test_world2_gloo_windows_and_split_frontier():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o[0])
    (_, s0, r0, b0, c0, p0, q0), (_, s1, r1, b1, c1, p1, q1) = outs
    # the split speculative solve is the reference's, pop for pop, on both ranks
    bw = _windows()[1]
    ref = orc.maximise_contrast_bnb(bw)
    assert p0 == p1 and p0[:4] == (ref.nu, ref.contrast, ref.bound_gap, ref.iterations)
    refc = orc.maximise_contrast_bnb(bw, max_iterations=4)
    assert q0 == q1 == (refc.nu, refc.contrast, 4)
    # both ranks hold the full, identical sample list and the identical BnB state
    assert s0 == s1 and r0 == r1
    # both ranks stop at the cap with the same incumbent
    assert c0 is not None and c0 == c1 and c0[2] == 3
    assert b0 and b1  # the broadcast window equals the source batch on both ranks
    serial = _oracle_stream(_windows(), SolverParams())
    assert s0 == [(s.t, s.contrast, s.iterations) for s in serial]
    # the split batched solve equals the single-process batched solve ...
    b = _windows()[1]
    c, bd = _oracle_evaluators(b)
    one = pdist.solve_batched(b, SolverParams(), k=8, contrasts=c, bounds=bd)
    assert (one.nu, one.contrast, one.rounds, one.nodes) == r0
    # ... and is certified within gamma of the reference-order optimum (P3)
    ref = orc.maximise_contrast_bnb(b)
    assert one.contrast >= ref.contrast - 0.025
    assert one.rounds <= ref.iterations


def test_batched_matches_reference_within_gamma_on_goldens(bnb_golden):
    meta, windows = bnb_golden
    for w, b in windows[:6]:
        c, bd = _oracle_evaluators(b)
        res = pdist.solve_batched(b, SolverParams(), k=16, contrasts=c, bounds=bd)
        ref_c = f64(w["result"]["contrast"])
        assert res.contrast >= ref_c - 0.025
        assert res.bound_gap <= 0.025 + 1e-12


def test_batched_iteration_cap_carries_incumbent():
    """solve_batched stops at params.max_iterations like solver.py:118-119:
    IterationLimitError carrying the incumbent after exactly that many nodes."""
    b = _windows()[1]
    c, bd = _oracle_evaluators(b)
    full = pdist.solve_batched(b, SolverParams(), k=4, contrasts=c, bounds=bd)
    assert full.nodes > 5
    for cap in (1, 5):
        with pytest.raises(IterationLimitError) as ei:
            pdist.solve_batched(b, SolverParams(max_iterations=cap), k=4, contrasts=c, bounds=bd)
        assert ei.value.iterations == cap
        assert ei.value.contrast <= full.contrast


@pytest.mark.parametrize("slots", [1, 3, 16])
def test_spec_solve_is_the_reference(bnb_golden, slots):
    """solve_spec replays the reference's pops exactly (nu, contrast,
    bound_gap and pop count bit-identical to the pinned oracle) for any number
    of speculative slots per round; more slots, fewer rounds."""
    meta, windows = bnb_golden
    rounds = []
    for w, b in windows[:6]:
        c, bd = _oracle_evaluators(b)
        r = pdist.solve_spec(b, SolverParams(), slots=slots, contrasts=c, bounds=bd)
        assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (
            f64(w["result"]["nu"]), f64(w["result"]["contrast"]), f64(w["result"]["bound_gap"]),
            w["result"]["iterations"])
        assert r.node_evals >= r.iterations - 1 and r.rounds <= r.iterations
        rounds.append((r.rounds, r.node_evals))
    if slots == 1:  # one node per round: the reference's own sequence of evaluations
        assert all(rd == ne for rd, ne in rounds)


def test_spec_solve_edges():
    """Iteration cap after the node that reaches it (incumbent carried), a
    root narrower than min_interval_width (its exact bound is the gap), and a
    window of one event."""
    b = _windows()[1]
    c, bd = _oracle_evaluators(b)
    for cap in (1, 2, 7):
        ref = orc.maximise_contrast_bnb(b, max_iterations=cap)
        if ref.status != "iteration_limit":
            continue
        with pytest.raises(IterationLimitError) as ei:
            pdist.solve_spec(b, SolverParams(max_iterations=cap), slots=5, contrasts=c, bounds=bd)
        assert (ei.value.nu, ei.value.contrast, ei.value.iterations) == (ref.nu, ref.contrast, cap)
    ref = orc.maximise_contrast_bnb(b, min_interval_width=3.0)
    r = pdist.solve_spec(b, SolverParams(min_interval_width=3.0), slots=4, contrasts=c, bounds=bd)
    assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (ref.nu, ref.contrast, ref.bound_gap,
                                                             ref.iterations)
    from paper_2209_13168_b200.events import EventBatch, SensorGeometry
    one = EventBatch(np.array([3.5]), np.array([2.25]), np.array([0.1]), 0.5, SensorGeometry(8, 6))
    c1, b1 = _oracle_evaluators(one)
    ref = orc.maximise_contrast_bnb(one)
    r = pdist.solve_spec(one, SolverParams(), slots=4, contrasts=c1, bounds=b1)
    assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (ref.nu, ref.contrast, ref.bound_gap,
                                                             ref.iterations)
