"""Median device time of evd_solve on configs 1-3 (and optionally 5).

python tools/time_solve.py [cfg ...]   -> one line per config
"""

import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import solver as sol, synth
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3]
    for c in cfgs:
        b = synth.config_window(c)
        ms = []
        for _ in range(5 if c != 5 else 2):
            r, st = sol.solve_window(b, evd.SolverParams())
            ms.append(st.device_ms)
        print(f"cfg {c}: n={b.n} iterations={r.iterations} device_ms median={statistics.median(ms):.3f} "
              f"min={min(ms):.3f}", flush=True)


if __name__ == "__main__":
    main()
