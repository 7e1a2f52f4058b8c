"""Benchmark: single-window BnB divergence solves on B200 (BASELINE.json configs[1]).

Workload (BASELINE.json configs[1], SURVEY.md §8(d) cfg 2): the 346x260
DAVIS-sized synthetic ventral-descent window, 204,203 events (window 0 of the
SimConfig(nu=-0.4, n_points=10000, seed=0) stream, regenerated bit-identically
by paper_2209_13168_b200.synth), one reference-order best-first BnB solve per
step (gamma=0.025, tau=0.5, epsilon=1e-6).

  value  solves/s with the window resident in HBM; device time of each step
         (CUDA events on the stream the persistent kernel runs on), L2 flushed
         between steps (the 4.9 MB window would otherwise stay in the 126 MB L2)
  e2e    the same metric through the public API maximise_contrast_bnb(batch)
         with pinned host arrays: per step H2D of the window + solve + D2H of
         the result, host wall clock
  --impl reference
         the reference algorithm's CPU implementation (the pinned oracle port,
         oracle/, every host thread) on the same window and metric; the stock
         numba reference (baseline/_ref/eventdiv, one core) is timed beside it
         once as cpu_baseline.reference_stock

Extra legs on the same line (each its own workload):
  solve_cfg3       cfg 3 (640x480, 999,557 events) single-window solve, device
                   and end to end (the north-star "~1M events in milliseconds")
  frontier_cfg3    the 4096-leaf frontier in one evd_eval_frontier call (tiled,
                   images in shared memory), with its own roofline
  windows_cfg4     2000-window landing sequence: one evd_solve_windows launch
                   (device), and end to end through
                   dist.estimate_stream_divergence_dist over the N ranks
                   (host batches in, every sample gathered on every rank)
  frontier_cfg5    cfg 5 (1280x720, 5.33 M events): the device-resident exact
                   solve, and dist.solve_batched_dist (event broadcast + the
                   batched frontier split over the N ranks)

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
(N>1: launch under torch.distributed.run; ranks solve independent windows.)
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = {"workload": "cfg2: 346x260 window, 204203 events, single-window BnB solve",
          "sensor": "346x260", "events": 204203, "gamma": 0.025, "tau": 0.5,
          "l2": "flushed between steps (256 MiB write)",
          "parallelism": "windows: one independent solve per rank (no data-path collective)"}
METRIC = "divergence solves/sec"
# cfg 2 runs the speculative-round solve (2 node evaluations per round; the
# library's policy for windows below 0.5M events on the whole grid)
KERNEL = "k_solve_spec"
UNIT = "solves/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML every 10 ms (nvidia-smi, ~0.5 s per call, as the fallback)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, {reason names})
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(device)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            try:
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device)
            bits = (pynvml.nvmlClocksEventReasonHwSlowdown,
                    pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwPowerCap)
            self._nvml = (pynvml, h, bits)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        pynvml, h, bits = self._nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        return sm, mx, {n for n, b in zip(self.NAMES, bits) if r & b}

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        v = [x.strip() for x in out.split(",")]
        if len(v) < 6 or not v[0].isdigit():
            return None
        return int(v[0]), int(v[1]) if v[1].isdigit() else None, \
            {n for n, x in zip(self.NAMES, v[2:]) if x.lower() == "active"}

    def _run(self):
        while not self._stop.is_set():
            try:
                s = self._sample_nvml() if self._nvml else self._sample_smi()
                if s:
                    self.samples.append(s)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples if s[1]]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def cpu_solve_sample(batch, threads):
    from oracle import oracle as orc
    orc.THREADS = threads
    t0 = time.perf_counter()
    r = orc.maximise_contrast_bnb(batch)
    return time.perf_counter() - t0, r


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def stock_reference(batch, timeout=600):
    """One cfg-2 maximise_contrast_bnb of the UNMODIFIED reference package
    (baseline/_ref/eventdiv: numpy + numba, single-threaded by construction),
    JIT warmed on a small window first, in a child process (its numba cache in
    /tmp).  Returns the cpu_baseline.reference_stock record."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "eventdiv")):
        return {"unavailable": "baseline/_ref/eventdiv not installed"}
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "w.npz")
        np.savez(path, x=batch.x, y=batch.y, t=batch.t)
        code = f"""
import json, sys, time
import numpy as np
sys.path.insert(0, {ref!r})
from eventdiv.events import EventBatch, SensorGeometry
from eventdiv.solver import SolverParams, maximise_contrast_bnb
z = np.load({path!r})
g = SensorGeometry({batch.geometry.width}, {batch.geometry.height})
r = np.random.default_rng(0)
w = EventBatch(r.uniform(0, 32, 300), r.uniform(0, 32, 300), np.sort(r.uniform(0, 0.5, 300)),
               0.5, SensorGeometry(32, 32))
maximise_contrast_bnb(w, SolverParams())   # numba JIT warm-up
b = EventBatch(z["x"], z["y"], z["t"], {float(batch.tau)!r}, g)
t0 = time.perf_counter()
res = maximise_contrast_bnb(b, SolverParams())
dt = time.perf_counter() - t0
print(json.dumps({{"s": dt, "nu": res.nu, "contrast": res.contrast, "iterations": res.iterations}}))
"""
        env = dict(os.environ, NUMBA_CACHE_DIR=os.path.join(tmp, "numba"),
                   PYTHONDONTWRITEBYTECODE="1", OMP_NUM_THREADS="1")
        try:
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                                 timeout=timeout, env=env)
            d = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception as e:
            return {"unavailable": f"stock reference run failed: {type(e).__name__}"}
    return {"value": 1.0 / d["s"], "unit": UNIT, "seconds_per_solve": d["s"], "cores": 1,
            "kind": "reference", "cpu": cpu_model(), "host_cores": host_threads(),
            "sample": "one full cfg-2 maximise_contrast_bnb of baseline/_ref/eventdiv "
                      "(numba JIT warmed; single-threaded by construction)",
            "result": {"nu": d["nu"], "contrast": d["contrast"], "iterations": d["iterations"]}}


def run_reference(args, rank, world):
    """The reference algorithm on the host cores (oracle port), rank 0 only."""
    if rank != 0:
        return
    from paper_2209_13168_b200 import synth
    batch = synth.config_window(2)
    threads = host_threads()
    for _ in range(args.warmup):
        cpu_solve_sample(batch, threads)
    times = []
    r = None
    for _ in range(args.steps):
        dt, r = cpu_solve_sample(batch, threads)
        times.append(dt)
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": CONFIG,
        "events_x_bound_evals_per_s": batch.n * r.bound_evals / (total / args.steps),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "one full cfg-2 BnB solve per step (96 iterations, 191 "
                                   "bound evals), oracle/ C restatement, events split over "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": {"nu": r.nu, "contrast": r.contrast, "iterations": r.iterations},
    }
    if not args.no_stock:
        line["cpu_baseline"]["reference_stock"] = stock_reference(batch)
    print(json.dumps(line), flush=True)


def load_json(*names):
    """The first of profiles/<name> that exists (newest round first)."""
    for n in names:
        f = os.path.join(ROOT, "profiles", n)
        if os.path.exists(f):
            with open(f) as fh:
                return json.load(fh), n
    return None, None


def ncu_val(nc, key):
    try:
        return float(str(nc[key][0]).replace(",", ""))
    except Exception:
        return None


def frontier_line(ctx, stream):
    """Config 3: the 4096-leaf frontier of a 999,557-event 640x480 window in one
    evd_eval_frontier call (device time, best of 3), tiled path (the 31 images
    of a work item in shared memory).  Roofline: shared-memory atomics, the
    marks (= upper_bound_image().in_image_events summed over the leaves) per
    second against the measured red.shared peak (tools/bench_fp64.cu)."""
    import torch
    from paper_2209_13168_b200 import contrast as con, frontier as fr, synth
    from paper_2209_13168_b200.geometry import velocity_domain
    b = synth.config_window(3)
    lo, hi = fr.uniform_frontier(velocity_domain(b.tau), 12)
    con.load_window(b, ctx)
    con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)  # bins the window (once per window)
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, _, mk = con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    info = ctx.frontier_info()
    marks = int(mk.sum())
    out = {"intervals": int(lo.size), "events": int(b.n), "seconds_per_call": best,
           "events_x_bound_evals_per_s": b.n * lo.size / best, "marks": marks,
           "path": {1: "tiles", 2: "global", 3: "global_exact"}.get(info["last_path"]),
           "tiles": info["tiles"], "listed_events": info["listed_events"]}
    peaks, _ = load_json("fp64_peak.json")
    nc, ncf = load_json("ncu_k_frontier_tiles_cfg3_r02.json")
    if peaks:
        # Binding roof: the fp64 division pipe.  The algorithm needs
        # one correctly rounded endpoint warp s = (1 + nu t) / (1 + nu tau) per
        # event and distinct endpoint -- K + 1 of them for a contiguous frontier
        # -- i.e. N (K + 1) IEEE quotients per call; achieved = that count per
        # second against the measured __ddiv_rn throughput.  (The kernel
        # certifies most of them from a reciprocal product instead of dividing.)
        pk = peaks.get("ddiv_rn_g_per_s")
        ach = b.n * (lo.size + 1) / best / 1e9
        spk = peaks.get("smem_red_u16pair_g_per_s")
        out["roofline"] = {
            "bound": "fp64_div", "kernel": "k_frontier_tiles", "achieved": ach, "peak": pk,
            "unit": "G quotients/s", "frac": ach / pk if pk else None,
            "traffic": nc.get("dram_bytes") if nc else None, "alg_bytes": 24 * b.n,
            "note": "achieved = events x (intervals + 1) endpoint warps per call / call time; "
                    "peak = __ddiv_rn throughput (profiles/fp64_peak.json, tools/bench_fp64.cu); "
                    "traffic = DRAM bytes of one call (ncu), the images never leave shared memory",
            "other_roofs": {"smem_atomic": {"achieved": marks / best / 1e9, "peak": spk,
                                            "unit": "G atomics/s",
                                            "frac": marks / best / 1e9 / spk if spk else None}}}
        if nc:
            out["limiter"] = {
                "kind": "issue / fp64 latency (certified filtered warps per event x interval)",
                "issue_active_pct": ncu_val(nc, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_pct": ncu_val(nc, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": ncu_val(nc, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                "source": f"profiles/{ncf}"}
    return out


def ref_loop_leg():
    """The reference's own BnB loop (baseline/_ref solver.py, Python heapq)
    with contrast_at / bound_terms bound to the drop-in,
    cfg 2, resident-window cache on and off (tools/ref_loop_bench.py)."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "eventdiv")):
        return {"unavailable": "baseline/_ref not installed (tools/install_reference.sh)"}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ref_loop_bench.py"), "2"],
                         capture_output=True, text=True, timeout=600)
    try:
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": (out.stderr or out.stdout)[-300:]}


def solve_leg(ctx, stream, flush, cfg, params, steps=5):
    """One single-window solve of config `cfg` per step: device time with the
    window resident (L2 flushed before each step), and end to end through
    maximise_contrast_bnb from pinned host arrays (H2D, solve, D2H)."""
    import torch
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import solver as sol, synth
    from paper_2209_13168_b200.contrast import load_window
    batch = synth.config_window(cfg)
    load_window(batch, ctx)
    res, _ = sol.solve_loaded(ctx, params)
    dev = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res, _ = sol.solve_loaded(ctx, params)
        e1.record(stream)
        torch.cuda.synchronize()
        dev.append(e0.elapsed_time(e1) / 1e3)
    pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(batch, k))).pin_memory()
           for k in ("x", "y", "t")}
    pb = evd.EventBatch(pin["x"].numpy(), pin["y"].numpy(), pin["t"].numpy(), batch.tau,
                        batch.geometry)
    evd.maximise_contrast_bnb(pb, params)
    e2e = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = evd.maximise_contrast_bnb(pb, params)
        e2e.append(time.perf_counter() - t0)
    return {"events": int(batch.n), "sensor": f"{batch.geometry.width}x{batch.geometry.height}",
            "device_ms": 1e3 * statistics.median(dev), "device_ms_min": 1e3 * min(dev),
            "e2e_ms": 1e3 * statistics.median(e2e), "solves_per_s": 1.0 / statistics.median(dev),
            "e2e_solves_per_s": 1.0 / statistics.median(e2e),
            "h2d_bytes": 24 * int(batch.n),
            "result": {"nu": res.nu, "contrast": res.contrast, "bound_gap": res.bound_gap,
                       "iterations": res.iterations, "bound_evals": res.bound_evals,
                       "device_rounds": int(res.rounds)},
            "same_as_public_api": (r.nu, r.contrast, r.iterations) ==
                                  (res.nu, res.contrast, res.iterations)}


def windows_line(ctx):
    """Config 4: the 2000-window 240x180 landing sequence in one evd_solve_windows
    launch (device time)."""
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import solver as sol, synth
    batches = [synth.sequence_window(k) for k in range(2000)]
    sol.solve_windows(batches[:64], evd.SolverParams(), ctx=ctx)
    # each mode: one warm-up call, then the median of 3 (wall clock, host batches in)
    def timed(overlap):
        ctx.set_option("stream_overlap", overlap)
        sol.solve_windows(batches, evd.SolverParams(), ctx=ctx)
        ts, out = [], None
        for _ in range(3):
            t0 = time.perf_counter()
            out = sol.solve_windows(batches, evd.SolverParams(), ctx=ctx)
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts), out
    # device time of the solve alone: upload first, then launch
    serial, (res, dev_s, groups) = timed(0)
    # the public path: the upload overlapped with the solve (evd_solve_windows_list)
    overlapped, (res2, _, _) = timed(1)
    same = [(r.nu, r.contrast, r.iterations) for r in res] == \
        [(r.nu, r.contrast, r.iterations) for r in res2]
    return {"windows": len(batches), "events": int(sum(b.n for b in batches)),
            "device_s": dev_s, "windows_per_s": len(batches) / dev_s, "solver_groups": groups,
            "e2e_s_upload_then_solve": serial, "e2e_s_overlapped": overlapped,
            "overlapped_identical": same,
            "all_ok": all(r.status == 0 for r in res)}, batches


def barrier_all(world):
    import torch
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()


def max_over_ranks(world, v):
    import torch
    if world == 1:
        return v
    tt = torch.tensor([v], device="cuda", dtype=torch.float64)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    return float(tt.item())


def windows_dist_leg(batches, world, reps=3):
    """Config 4 end to end on N ranks: dist.estimate_stream_divergence_dist over
    the 2000 host windows -- every rank copies its contiguous shard (balanced
    by events) to its GPU, solves it in one launch and the per-window samples
    are all-gathered; wall time between barriers, max over ranks (fixed total
    work: strong scaling)."""
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import dist as pdist
    params = evd.SolverParams()
    out = pdist.estimate_stream_divergence_dist(batches, params)  # warm-up
    best = None
    for _ in range(reps):
        barrier_all(world)
        t0 = time.perf_counter()
        out = pdist.estimate_stream_divergence_dist(batches, params)
        barrier_all(world)
        t = max_over_ranks(world, time.perf_counter() - t0)
        best = t if best is None else min(best, t)
    return {"windows": len(batches), "ranks": world, "e2e_s": best,
            "windows_per_s": len(batches) / best, "samples": len(out),
            "h2d_bytes": 24 * int(sum(b.n for b in batches)),
            "scaling": "strong (2000 windows split over the ranks)"}


def cfg5_leg(world, rank):
    """Config 5 (1280x720, 5,327,641 events): the single-GPU device-resident
    exact solve (maximise_contrast_bnb), dist.solve_batched_dist on the N
    ranks (events broadcast once over NCCL, each round's evaluations split
    over the ranks, results all-gathered; certified within gamma) and
    dist.solve_spec_dist (the same split, replaying the reference's pops
    exactly)."""
    import torch
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import dist as pdist, synth
    params = evd.SolverParams()
    batch = synth.config_window(5) if rank == 0 else None
    out = {"events": 5327641, "sensor": "1280x720", "ranks": world}
    if rank == 0:
        evd.maximise_contrast_bnb(batch, params)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = evd.maximise_contrast_bnb(batch, params)
        out["exact_solve_e2e_s"] = time.perf_counter() - t0
        out["exact"] = {"nu": r.nu, "contrast": r.contrast, "iterations": r.iterations}
    pdist.solve_batched_dist(batch, params, k=64)  # warm-up (broadcast + evaluators)
    barrier_all(world)
    t0 = time.perf_counter()
    rb = pdist.solve_batched_dist(batch, params, k=64)
    barrier_all(world)
    out["batched_dist_e2e_s"] = max_over_ranks(world, time.perf_counter() - t0)
    out["batched"] = {"nu": rb.nu, "contrast": rb.contrast, "rounds": rb.rounds,
                      "nodes": rb.nodes, "bound_evals": rb.bound_evals, "k": 64}
    if rank == 0:
        out["batched_within_gamma"] = rb.contrast >= out["exact"]["contrast"] - params.gamma
    # the exact speculative split solve: the reference's pops, each round's
    # node evaluations (4 per rank) split over the ranks
    pdist.solve_spec_dist(batch, params, slots_per_rank=4)  # warm-up
    barrier_all(world)
    t0 = time.perf_counter()
    rs = pdist.solve_spec_dist(batch, params, slots_per_rank=4)
    barrier_all(world)
    out["spec_dist_e2e_s"] = max_over_ranks(world, time.perf_counter() - t0)
    out["spec_dist"] = {"nu": rs.nu, "contrast": rs.contrast, "iterations": rs.iterations,
                        "rounds": rs.rounds, "node_evals": rs.node_evals,
                        "slots": 4 * world}
    if rank == 0:
        out["spec_dist_identical"] = (rs.nu, rs.contrast, rs.iterations) == (
            r.nu, r.contrast, r.iterations)
    return out


def stream_line():
    """Whole-stream pipeline end to end (tools/bench_stream.py): 50 landing
    descents at 240x180 as one stream and as one EVD1 file."""
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_stream.py"), "50"],
                         capture_output=True, text=True, timeout=600)
    try:
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": (out.stderr or out.stdout)[-300:]}


def run_gpu(args, rank, world, local):
    import torch
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import _lib, contrast, solver as sol, synth
    from paper_2209_13168_b200.contrast import load_window

    # End-to-end legs copy each step's window host -> device: the per-call
    # resident-window cache (contrast.load_window) would skip that copy when
    # the same host arrays come back, so it is off for the whole benchmark
    # (the reference_loop_drop_in leg measures it separately, in its own process).
    contrast.WINDOW_CACHE = False

    torch.cuda.set_device(local)
    _lib.set_device(local)
    import torch.distributed as dist
    if world == 1 and not args.no_extra:
        # a one-rank NCCL group, so the multi-GPU legs run their real code path
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(port))
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    elif world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    batch = synth.config_window(2)
    params = evd.SolverParams()
    ctx = _lib.context(local)
    # one explicit stream for the library, the flush and the timing events
    # (torch's default stream has handle 0, which evd_set_stream reads as
    # "the context's own stream")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.lib.evd_set_stream(ctx.h, _lib._vp(stream.cuda_stream))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---------------- value: resident window, device-timed steps
    load_window(batch, ctx)
    for _ in range(args.warmup):
        res, _ = sol.solve_loaded(ctx, params)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kernel_ms = []
    barrier()
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            res, _ = sol.solve_loaded(ctx, params)
            ev[k][1].record(stream)
            kernel_ms.append(res.device_ms)
        barrier()
    launches = ctx.launches - launches0
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    t_dev = dev_ms / 1e3
    if world > 1:
        tt = torch.tensor([t_dev], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_dev = float(tt.item())
    value = world * args.steps / t_dev

    # ---------------- e2e: public API, pinned host buffers, H2D + solve + D2H each step
    pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(batch, k))).pin_memory()
           for k in ("x", "y", "t")}
    pbatch = evd.EventBatch(pin["x"].numpy(), pin["y"].numpy(), pin["t"].numpy(), batch.tau,
                            batch.geometry)
    for _ in range(args.warmup):
        evd.maximise_contrast_bnb(pbatch, params)
    barrier()
    t_e2e = 0.0
    for _ in range(args.steps):
        flush.zero_()  # same L2 state as the device-timed leg, outside the timed call
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = evd.maximise_contrast_bnb(pbatch, params)  # synchronous: H2D, solve, D2H
        t_e2e += time.perf_counter() - t0
    barrier()
    if world > 1:
        tt = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e = world * args.steps / t_e2e

    # ---------------- extra legs (all ranks take part in the multi-rank ones)
    extra = {}
    if not args.no_extra:
        if world == 1:
            extra["frontier_cfg3"] = frontier_line(ctx, stream)
            extra["solve_cfg3"] = solve_leg(ctx, stream, flush, 3, params)
            wl, batches = windows_line(ctx)
            extra["windows_cfg4"] = wl
        else:
            from paper_2209_13168_b200 import synth as _s
            batches = [_s.sequence_window(k) for k in range(2000)]
        extra["windows_cfg4_dist"] = windows_dist_leg(batches, world)
        extra["frontier_cfg5"] = cfg5_leg(world, rank)
        if world == 1:
            extra["stream_e2e"] = stream_line()
            extra["reference_loop_drop_in"] = ref_loop_leg()

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                peaks = json.load(fh)
        except Exception:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        k_ms = statistics.mean(kernel_ms)
        # Node evaluations the kernel actually executed, speculative slots
        # included: every evaluation passes over all n events (exact_events)
        node_evals = int(round(res.exact_events / batch.n))
        nc, ncf = load_json("ncu_k_solve_cfg2_r02.json", "ncu_k_solve_cfg2_r01.json")
        traffic = nc.get("dram_bytes") if nc and "dram_bytes" in nc else None
        if nc and traffic is None:
            tb = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic = int(sum(ncu_val(nc, k) * tb.get(nc[k][1], 1)
                              for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")))
        # binding roof of k_solve_spec: every pixel increment is one L2 RED
        # (explicit red.global), marks = the reference's in_image_events summed
        # over the solve's images; peak measured by tools/bench_atomics.cu at
        # this image size (profiles/atomic_peak.json).  HBM is not binding: the
        # window is L2-resident, DRAM traffic is below the algorithmic bytes.
        apk_all, _ = load_json("atomic_peak.json")
        apk = (apk_all or {}).get("random_m89960_gatomics_per_s")
        ach = res.marks / (k_ms / 1e3) / 1e9
        alg_bytes = 24.0 * batch.n * node_evals
        hbm_ach = alg_bytes / (k_ms / 1e3) / 1e9
        fp64pk, _ = load_json("fp64_peak.json")
        limiter = None
        if nc:
            limiter = {
                "kind": "latency / issue (sequential BnB rounds; per-warp dependent chains)",
                "atomic_roof_binding": False,
                "atomic_evidence": "profiles/no_red_ab_r02.txt: segment REDs compiled out "
                                   "(-DEVD_NO_RED) change the event pass by <= 1% at the cfg-2 "
                                   "root (144.0 -> 143.2 us) and narrow nodes (10.2 -> 10.0 us)",
                "issue_active_pct": ncu_val(nc, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": ncu_val(nc, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_pct": ncu_val(nc, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                "threads_per_warp_inst": ncu_val(nc, "smsp__thread_inst_executed_per_inst_executed.ratio"),
                "registers_per_thread": ncu_val(nc, "launch__registers_per_thread"),
                "source": f"profiles/{ncf}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference simulator restated, bit-identical window)",
            "config": CONFIG,
            "events_x_bound_evals_per_s": world * batch.n * res.bound_evals * args.steps / t_dev,
            "solve": {"nu": res.nu, "contrast": res.contrast, "bound_gap": res.bound_gap,
                      "iterations": res.iterations, "bound_evals": res.bound_evals,
                      "point_evals": res.point_evals, "node_evals": node_evals,
                      "max_frontier": res.max_frontier, "marks": int(res.marks),
                      "kernel_ms": k_ms, "device_rounds": int(res.rounds)},
            # per step: x, y, t (f64) and the window offsets in; one WindowResult
            # (evd_internal.h) out
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 24 * batch.n + 16,
                    "d2h_bytes_per_step": ctypes.sizeof(_lib.WindowResult)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "roofline": {"bound": "atomic", "kernel": KERNEL, "achieved": ach, "peak": apk,
                         "unit": "G atomics/s", "frac": ach / apk if apk else None,
                         "traffic": traffic, "marks_per_launch": int(res.marks),
                         "note": "achieved = marks per solve (sum of every image's "
                                 "in_image_events) / mean kernel time; peak = u32 RED at "
                                 "M=89,960 (tools/bench_atomics.cu); traffic = DRAM bytes of "
                                 "one launch (ncu --set full)",
                         "other_roofs": {
                             "hbm": {"achieved": hbm_ach, "peak": hbm_peak, "unit": "GB/s",
                                     "frac": hbm_ach / hbm_peak,
                                     "alg_bytes": alg_bytes,
                                     "note": "24 B x events x node evaluations; the window is "
                                             "L2-resident"},
                             "fp64_pipe_pct": limiter["fp64_pipe_pct"] if limiter else None,
                             "fp64_peaks": fp64pk}},
            "limiter": limiter,
        }
        line.update(extra)
        if world == 1 and not args.no_cpu:
            threads = host_threads()
            dt, r = cpu_solve_sample(batch, threads)
            same = (r.nu, r.contrast, r.iterations) == (res.nu, res.contrast, res.iterations)
            line["cpu_baseline"] = {
                "value": 1.0 / dt, "unit": UNIT, "cores": threads, "kind": "port",
                "cpu": cpu_model(),
                "sample": "one full cfg-2 BnB solve (oracle/ C restatement of the reference, "
                          f"events split over {threads} threads); identical result: {same}"}
            if not args.no_stock:
                line["cpu_baseline"]["reference_stock"] = stock_reference(batch)
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the config-3/4/5 legs")
    ap.add_argument("--no-stock", action="store_true",
                    help="skip timing the stock numba reference (baseline/_ref)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_gpu(args, rank, world, local)


if __name__ == "__main__":
    main()
