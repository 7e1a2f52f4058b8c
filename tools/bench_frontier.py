"""Throughput of the batched frontier (config 3: 640x480 window, 999,557 events,
the 4096 depth-12 leaves of the root bisection in one evd_eval_frontier call).

python tools/bench_frontier.py [reps] [path]   -> one JSON line
path: auto (default) | tiles | global | global_exact | per_interval (evd_set_option "frontier_path")
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2209_13168_b200 import _lib, contrast as con, frontier as fr, synth
    from paper_2209_13168_b200.geometry import velocity_domain

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    b = synth.config_window(3)
    lo, hi = fr.uniform_frontier(velocity_domain(b.tau), 12)
    ctx = _lib.context()
    path = sys.argv[2] if len(sys.argv) > 2 else "auto"
    ctx.set_option("frontier_path", {"auto": 0, "tiles": 1, "global": 2, "global_exact": 3,
                                     "per_interval": 4}[path])
    stream = torch.cuda.Stream()  # explicit: handle 0 would mean the context's own stream
    torch.cuda.set_stream(stream)
    ctx.lib.evd_set_stream(ctx.h, _lib._vp(stream.cuda_stream))
    con.load_window(b, ctx)
    for _ in range(2):
        s, fi, mk = con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)
    times = []
    l0 = ctx.launches
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        s, fi, mk = con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    launches = (ctx.launches - l0) // reps
    t = min(times)
    units = b.n * lo.size
    marks = int(mk.sum())
    apk = None
    afile = os.path.join(ROOT, "profiles", "atomic_peak.json")
    if os.path.exists(afile):
        with open(afile) as fh:
            apk = json.load(fh).get("random_m307200_gatomics_per_s")
    print(json.dumps({
        "workload": "cfg3 frontier: 640x480, %d events, %d intervals per call" % (b.n, lo.size),
        "seconds_per_call": t, "median_s": float(np.median(times)),
        "events_x_bound_evals_per_s": units / t,
        "marks": marks, "marks_per_event_interval": marks / units,
        "checksum": [int(s.astype(np.uint64).sum(dtype=np.uint64)), int(fi.sum())],
        "atomics_per_s": marks / t, "atomic_peak": apk,
        "atomic_frac": (marks / t / 1e9 / apk) if apk else None,
        "launches_per_call": launches, "path": path, "info": ctx.frontier_info(),
        "hbm_alg_bytes": 24 * b.n, "note": "events read once per call (24 B/event)",
    }))


if __name__ == "__main__":
    main()
