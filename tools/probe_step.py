"""Sub-phases of the speculative round's replicated step (experiment build
with -DEVD_TRACE_BUILD -DEVD_STEP_PROBE): per round, step start -> results
inserted -> pops done -> step end (us, block 0).

EVD_LIB=build_var/probe_trace.so python tools/probe_step.py [cfg]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["EVD_TRACE"] = "1"
os.environ["EVD_TRACE_SPEC"] = "1"

import paper_2209_13168_b200 as evd  # noqa: E402
from paper_2209_13168_b200 import _lib, solver as sol, synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    b = synth.config_window(cfg)
    for _ in range(3):
        r, st = sol.solve_window(b, evd.SolverParams())
    ctx = _lib.context()
    buf = np.zeros(1 + 10 * (1 << 14), dtype=np.int64)
    n = np.zeros(1, dtype=np.int64)
    ctx.lib.evd_solve_trace(ctx.h, _lib.ptr(buf, _lib._i64p), buf.size, _lib.ptr(n, _lib._i64p))
    res, _ = sol.solve_loaded(ctx, evd.SolverParams())
    k = res.rounds
    raw = buf[1:1 + 10 * k].reshape(k, 10).astype(np.float64) / 1e3
    ins = raw[:, 8] - raw[:, 6]
    pops = raw[:, 9] - raw[:, 8]
    sel = raw[:, 7] - raw[:, 9]
    print(f"cfg {cfg}: rounds {k}; step sub-phases (us, median / sum): "
          f"results+insert {np.median(ins[:-1]):.1f} / {ins[:-1].sum():.0f}, "
          f"pops {np.median(pops[:-1]):.1f} / {pops[:-1].sum():.0f}, "
          f"selection {np.median(sel[:-1]):.1f} / {sel[:-1].sum():.0f}")


if __name__ == "__main__":
    main()
