"""Throughput of many-window solves (config 4: the 2000-window 240x180 landing
sequence of SURVEY §8(d)), one evd_solve_windows launch.

python tools/bench_windows.py [n_windows] [groups ...]   -> JSON lines
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import solver as sol, synth

    nw = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    groups = [int(g) for g in sys.argv[2:]] or [0]
    t0 = time.perf_counter()
    batches = [synth.sequence_window(k) for k in range(nw)]
    gen = time.perf_counter() - t0
    ev = sum(b.n for b in batches)
    for g in groups:
        sol.solve_windows(batches[: min(nw, 64)], evd.SolverParams(), groups=g)  # warm
        t0 = time.perf_counter()
        res, dev_s, used = sol.solve_windows(batches, evd.SolverParams(), groups=g)
        wall = time.perf_counter() - t0
        evals = sum(int(r.bound_evals) for r in res)
        print(json.dumps({
            "workload": f"cfg4: {nw} windows 240x180, {ev} events", "groups": used,
            "device_s": dev_s, "wall_s": wall, "windows_per_s": nw / dev_s,
            "e2e_windows_per_s": nw / wall,
            "events_x_bound_evals_per_s": sum(b.n * int(r.bound_evals) for b, r in
                                              zip(batches, res)) / dev_s,
            "bound_evals": evals, "gen_s": gen,
            "all_ok": all(r.status == 0 for r in res)}), flush=True)


if __name__ == "__main__":
    main()
