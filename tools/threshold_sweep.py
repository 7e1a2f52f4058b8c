"""Solve time vs window size for each CTA size / slot count (policy thresholds
kSmallWindow / kLargeWindow / kSpecMaxEvents in csrc/evd_api.cu).

python tools/threshold_sweep.py  -> one line per (n, block, spec)
"""

import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(n, cfg):
    import numpy as np
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import solver as sol, synth
    from paper_2209_13168_b200.events import EventBatch
    b = synth.config_window(cfg)
    idx = np.sort(np.random.default_rng(n).choice(b.n, size=min(n, b.n), replace=False))
    w = EventBatch(b.x[idx], b.y[idx], b.t[idx], b.tau, b.geometry)
    ms = []
    for _ in range(5):
        r, st = sol.solve_window(w, evd.SolverParams())
        ms.append(st.device_ms)
    print(f"n={w.n} block={os.environ.get('EVD_SOLVE_BLOCK')} spec={os.environ.get('EVD_SPEC_K')} "
          f"ms={statistics.median(ms):.3f}", flush=True)


def main():
    if len(sys.argv) > 2:
        return child(int(sys.argv[1]), int(sys.argv[2]))
    for n, cfg in ((50000, 2), (100000, 2), (150000, 2), (400000, 3), (700000, 3)):
        for blk in (384, 512, 768):
            for k in (1, 3, 4):
                env = dict(os.environ, EVD_SOLVE_BLOCK=str(blk), EVD_SPEC_K=str(k))
                subprocess.run([sys.executable, __file__, str(n), str(cfg)], env=env)


if __name__ == "__main__":
    main()
