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
         oracle/, every host thread) on the same window and metric

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
          "l2": "flushed between steps (256 MiB write)"}
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
    print(json.dumps(line), flush=True)


def frontier_line(ctx, stream):
    """Config 3: the 4096-leaf frontier of a 999,557-event 640x480 window in one
    evd_eval_frontier call (device time, best of 3)."""
    import torch
    from paper_2209_13168_b200 import contrast as con, frontier as fr, synth
    from paper_2209_13168_b200.geometry import velocity_domain
    b = synth.config_window(3)
    lo, hi = fr.uniform_frontier(velocity_domain(b.tau), 12)
    con.load_window(b, ctx)
    con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, _, mk = con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    return {"intervals": int(lo.size), "events": int(b.n), "seconds_per_call": best,
            "events_x_bound_evals_per_s": b.n * lo.size / best,
            "marks": int(mk.sum()), "atomics_per_s": float(mk.sum()) / best}


def windows_line(ctx):
    """Config 4: the 2000-window 240x180 landing sequence in one evd_solve_windows
    launch (device time)."""
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import solver as sol, synth
    batches = [synth.sequence_window(k) for k in range(2000)]
    sol.solve_windows(batches[:64], evd.SolverParams(), ctx=ctx)
    res, dev_s, groups = sol.solve_windows(batches, evd.SolverParams(), ctx=ctx)
    return {"windows": len(batches), "events": int(sum(b.n for b in batches)),
            "device_s": dev_s, "windows_per_s": len(batches) / dev_s, "solver_groups": groups,
            "all_ok": all(r.status == 0 for r in res)}


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
    from paper_2209_13168_b200 import _lib, solver as sol, synth
    from paper_2209_13168_b200.contrast import load_window

    torch.cuda.set_device(local)
    _lib.set_device(local)
    if world > 1:
        import torch.distributed as dist
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

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                peaks = json.load(fh)
        except Exception:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        # algorithmic bytes of k_solve: each node evaluation streams the window
        # once (24 B/event: x, y, t); images are not algorithmic
        alg_bytes = 24.0 * batch.n * res.point_evals
        k_ms = statistics.mean(kernel_ms)
        achieved = alg_bytes / (k_ms / 1e3) / 1e9
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tfile):
            with open(tfile) as fh:
                traffic = json.load(fh).get("k_solve_dram_bytes")
        # atomic roofline: every pixel increment is one L2 RED; peak measured by
        # tools/bench_atomics.cu for this image size (profiles/atomic_peak.json)
        atomic = None
        afile = os.path.join(ROOT, "profiles", "atomic_peak.json")
        if os.path.exists(afile):
            with open(afile) as fh:
                apk = json.load(fh).get("random_m89960_gatomics_per_s")
            ach = res.marks / (k_ms / 1e3) / 1e9
            atomic = {"achieved": ach, "peak": apk, "unit": "G atomics/s",
                      "frac": ach / apk if apk else None, "marks_per_solve": int(res.marks),
                      "peak_source": "tools/bench_atomics.cu (u32 RED, random pixels, M=89960)"}
        # what does bound the kernel: issue and occupancy from the committed
        # ncu --set full capture of this launch (profiles/, tools/round_evidence.sh)
        limiter = None
        nfile = os.path.join(ROOT, "profiles", "ncu_k_solve_cfg2_r01.json")
        if os.path.exists(nfile):
            with open(nfile) as fh:
                nc = json.load(fh)
            g = lambda k: float(nc[k][0]) if k in nc else None
            limiter = {
                "kind": "latency / issue (sequential BnB rounds; per-warp dependent chains)",
                "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_pct": g("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                "threads_per_warp_inst": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
                "registers_per_thread": g("launch__registers_per_thread"),
                "source": "profiles/ncu_k_solve_cfg2_r01.json"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference simulator restated, bit-identical window)",
            "config": dict(CONFIG, parallelism=f"windows x{world} (no data-path collective)"),
            "events_x_bound_evals_per_s": world * batch.n * res.bound_evals * args.steps / t_dev,
            "solve": {"nu": res.nu, "contrast": res.contrast, "bound_gap": res.bound_gap,
                      "iterations": res.iterations, "bound_evals": res.bound_evals,
                      "point_evals": res.point_evals, "max_frontier": res.max_frontier,
                      "marks": int(res.marks), "kernel_ms": k_ms,
                      "device_rounds": int(res.rounds)},
            "atomic_roofline": atomic,
            "limiter": limiter,
            # per step: x, y, t (f64) and the window offsets in; one WindowResult
            # (evd_internal.h) out
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 24 * batch.n + 16,
                    "d2h_bytes_per_step": ctypes.sizeof(_lib.WindowResult)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "roofline": {"bound": "hbm", "kernel": KERNEL, "achieved": achieved,
                         "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                         "traffic": traffic,
                         "note": "latency-bound sequential BnB: grid-wide rounds of node "
                                 "evaluations; algorithmic bytes = 24 B x events x node evals"},
        }
        if world == 1 and not args.no_extra:
            line["frontier_cfg3"] = frontier_line(ctx, stream)
            line["windows_cfg4"] = windows_line(ctx)
            line["stream_e2e"] = stream_line()
        if world == 1 and not args.no_cpu:
            threads = host_threads()
            dt, r = cpu_solve_sample(batch, threads)
            same = (r.nu, r.contrast, r.iterations) == (res.nu, res.contrast, res.iterations)
            line["cpu_baseline"] = {
                "value": 1.0 / dt, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": "one full cfg-2 BnB solve (oracle/ C restatement of the reference, "
                          f"events split over {threads} threads); identical result: {same}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the config-3 frontier and config-4 window lines")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_gpu(args, rank, world, local)


if __name__ == "__main__":
    main()
