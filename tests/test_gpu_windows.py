"""Many windows per launch (evd_solve_windows) == one solve per window (GPU)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, f64
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import _lib, solver as sol, synth
from paper_2209_13168_b200.events import EventBatch, SensorGeometry

pytestmark = pytest.mark.gpu


def _same(r, ref):
    return (r.nu, r.contrast, r.bound_gap, int(r.iterations)) == (
        f64(ref["nu"]), f64(ref["contrast"]), f64(ref["bound_gap"]), ref["iterations"])


@pytest.mark.parametrize("groups", [0, 1, 3, 7, 74, 148])
def test_sequence_windows_match_reference(groups):
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        seq = json.load(fh)["sequence"]
    batches = [synth.sequence_window(s["k"]) for s in seq]
    res, secs, g = sol.solve_windows(batches, evd.SolverParams(), groups=groups)
    assert secs > 0 and g >= 1
    for r, s in zip(res, seq):
        assert r.status == 0 and _same(r, s["result"]), (s["k"], r.nu)


def test_small_windows_and_gaps(bnb_golden):
    meta, windows = bnb_golden
    g = SensorGeometry(64, 64)
    picks = [(w, b) for w, b in windows if b.geometry.width == 64 and b.geometry.height == 64]
    empty = EventBatch(np.empty(0), np.empty(0), np.empty(0), 0.5, g)
    batches = [picks[0][1], empty] + [b for _, b in picks[1:]]
    res, _, _ = sol.solve_windows(batches, evd.SolverParams(), groups=2)
    assert res[1].status == _lib.EVD_ERR_NO_EVENTS
    live = [r for j, r in enumerate(res) if j != 1]
    for r, (w, _) in zip(live, picks):
        assert r.status == 0 and _same(r, w["result"])


def test_iteration_limit_per_window(bnb_golden):
    meta, windows = bnb_golden
    lim = meta["iteration_limit"]
    b = windows[lim["window"]][1]
    res, _, _ = sol.solve_windows([b, b], evd.SolverParams(max_iterations=lim["max_iterations"]),
                                  groups=2)
    for r in res:
        assert r.status == _lib.EVD_ERR_ITER_LIMIT
        assert (r.nu, r.contrast, int(r.iterations)) == (f64(lim["nu"]), f64(lim["contrast"]),
                                                         lim["iterations"])


def test_stream_driver_matches_per_window():
    batches = [synth.sequence_window(k) for k in (10, 11, 12, 13)]
    samples = evd.estimate_stream_divergence(batches, evd.SolverParams())
    for s, b in zip(samples, batches):
        r = evd.maximise_contrast_bnb(b, evd.SolverParams())
        assert (s.contrast, s.iterations) == (r.contrast, r.iterations)
        assert s.divergence == evd.divergence_from_velocity(r.nu, b.tau)


@pytest.mark.parametrize("cfg,k", [("1", 16), ("2", 64)])
def test_batched_frontier_bnb_within_gamma(cfg, k):
    """Batched best-first (k nodes per round, one frontier pass per round) on
    the GPU: certified within gamma of the reference optimum (parity P3)."""
    from paper_2209_13168_b200 import dist as pdist
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        ref = json.load(fh)["configs"][cfg]["result"]
    b = synth.config_window(int(cfg))
    r = pdist.solve_batched(b, evd.SolverParams(), k=k)
    assert r.contrast >= f64(ref["contrast"]) - 0.025
    assert r.bound_gap <= 0.025
    assert r.rounds < ref["iterations"]
    # the incumbent is a real contrast value of the reference objective
    assert r.contrast == evd.contrast_at(b, r.nu)


def test_dist_batched_over_nccl_world1():
    """The multi-GPU frontier path on one GPU: events broadcast over NCCL and
    loaded from device memory, results gathered as tensors; equals the
    single-process batched solve."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2209_13168_b200 import dist as pdist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        b = synth.config_window(1)
        got = pdist.solve_batched_dist(b, evd.SolverParams(), k=16)
    finally:
        dist.destroy_process_group()
    ref = pdist.solve_batched(b, evd.SolverParams(), k=16)
    assert (got.nu, got.contrast, got.bound_gap, got.rounds, got.nodes) == (
        ref.nu, ref.contrast, ref.bound_gap, ref.rounds, ref.nodes)


@pytest.mark.parametrize("cfg", [1, 2])
def test_spec_dist_solve_is_the_reference(cfg):
    """dist.solve_spec_dist (NCCL broadcast, libevd evaluators from device
    memory, speculative rounds) gives the reference's BnbResult, pop count
    included, at configs 1 and 2."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2209_13168_b200 import dist as pdist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        b = synth.config_window(cfg)
        got = pdist.solve_spec_dist(b, evd.SolverParams(), slots_per_rank=6)
    finally:
        dist.destroy_process_group()
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        ref = json.load(fh)["configs"][str(cfg)]["result"]
    assert (got.nu, got.contrast, got.bound_gap, got.iterations) == (
        f64(ref["nu"]), f64(ref["contrast"]), f64(ref["bound_gap"]), ref["iterations"])


@pytest.mark.parametrize("chunk", [1024, 7000, 1 << 16])
def test_windows_list_overlapped_upload(chunk):
    """evd_solve_windows_list: the solve starts before the host windows are
    uploaded (chunks spanning window boundaries, an empty window between);
    results and the resident window set afterwards equal upload-then-solve."""
    import ctypes
    g = SensorGeometry(240, 180)
    batches = [synth.sequence_window(k) for k in range(20, 29)]
    batches.insert(4, EventBatch(np.empty(0), np.empty(0), np.empty(0), batches[0].tau, g))
    ctx = _lib.Context(0)

    def resident():
        out = [np.zeros(1, dtype=np.uint64), np.zeros(1, dtype=np.int64),
               np.zeros(1, dtype=np.uint64)]
        lo, hi = np.array([-1.5]), np.array([-0.3])
        rc = ctx.lib.evd_bound_images(ctx.h, _lib.ptr(lo), _lib.ptr(hi), 1,
                                      _lib.ptr(out[0], _lib._u64p), _lib.ptr(out[1], _lib._i64p),
                                      _lib.ptr(out[2], _lib._u64p),
                                      ctypes.POINTER(ctypes.c_uint32)())
        assert rc == 0
        return [int(a[0]) for a in out]

    ctx.set_option("stream_overlap", 0)
    want, _, _ = sol.solve_windows(batches, evd.SolverParams(), ctx=ctx)
    want_res = resident()
    ctx.set_option("stream_overlap", 1)
    ctx.set_option("stream_chunk", chunk)
    got, secs, _ = sol.solve_windows(batches, evd.SolverParams(), ctx=ctx)
    assert secs > 0
    key = lambda rs: [(r.status, r.nu, r.contrast, r.bound_gap, r.iterations) for r in rs]
    assert key(got) == key(want)
    assert got[4].status == _lib.EVD_ERR_NO_EVENTS
    assert resident() == want_res
    # every window empty: no solve, statuses only
    empties = [batches[4]] * 3
    res, _, _ = sol.solve_windows(empties, evd.SolverParams(), ctx=ctx)
    assert all(r.status == _lib.EVD_ERR_NO_EVENTS for r in res)
