"""Same-box A/B of the resident-window solve (evd_solve, device time) and the
end-to-end maximise_contrast_bnb from pinned host arrays, per library:

EVD_LIB=build_var/X.so python tools/ab_e2e.py [cfg ...]
"""
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import contrast, solver as sol, synth
    for cfg in [int(a) for a in sys.argv[1:]] or [1, 2, 3]:
        b = synth.config_window(cfg)
        pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory() for k in "xyt"}
        pb = evd.EventBatch(pin["x"].numpy(), pin["y"].numpy(), pin["t"].numpy(), b.tau, b.geometry)
        p = evd.SolverParams()
        dev, e2e = [], []
        for i in range(12):
            ctx = contrast.load_window(b, cache=False)
            res, _ = sol.solve_loaded(ctx, p)
            dev.append(res.device_ms)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = evd.maximise_contrast_bnb(pb, p)
            e2e.append(1e3 * (time.perf_counter() - t0))
        print(f"cfg {cfg}: resident solve {statistics.median(dev[2:]):.3f} ms, "
              f"maximise_contrast_bnb (pinned) {statistics.median(e2e[2:]):.3f} ms, "
              f"nu={r.nu!r} it={r.iterations}", flush=True)


if __name__ == "__main__":
    main()
