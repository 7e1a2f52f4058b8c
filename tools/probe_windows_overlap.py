"""Config 4 (2000 windows, 240x180) through solve_windows with the upload
overlapped (evd_solve_windows_list) and without; wall time per call, median
of 3 after a warm-up; results must be identical.

python tools/probe_windows_overlap.py
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import _lib, solver as sol, synth
    batches = [synth.sequence_window(k) for k in range(2000)]
    ctx = _lib.context()
    params = evd.SolverParams()
    sol.solve_windows(batches[:64], params, ctx=ctx)
    key0 = None
    for overlap, chunk in ((0, 0), (1, 1 << 15), (1, 1 << 16), (1, 1 << 17), (0, 0)):
        ctx.set_option("stream_overlap", overlap)
        if chunk:
            ctx.set_option("stream_chunk", chunk)
        ts, dev = [], []
        for _ in range(4):
            t0 = time.perf_counter()
            res, d, g = sol.solve_windows(batches, params, ctx=ctx)
            ts.append(time.perf_counter() - t0)
            dev.append(d)
        key = [(r.nu, r.contrast, r.iterations) for r in res]
        key0 = key0 or key
        print(f"overlap={overlap} chunk={chunk}: wall {1e3 * statistics.median(ts[1:]):.1f} ms, "
              f"device {1e3 * statistics.median(dev[1:]):.1f} ms, groups {g}, "
              f"same={key == key0}", flush=True)


if __name__ == "__main__":
    main()
