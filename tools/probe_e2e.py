"""Host-side breakdown of one end-to-end cfg-2 solve (maximise_contrast_bnb
from pinned host arrays): upload, solve call, total.

python tools/probe_e2e.py [cfg]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import contrast, solver as sol, synth
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    b = synth.config_window(cfg)
    pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory() for k in "xyt"}
    pb = evd.EventBatch(pin["x"].numpy(), pin["y"].numpy(), pin["t"].numpy(), b.tau, b.geometry)
    p = evd.SolverParams()
    for _ in range(3):
        evd.maximise_contrast_bnb(pb, p)
    up, so, tot, dev = [], [], [], []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx = contrast.load_window(pb, cache=False)
        t1 = time.perf_counter()
        res, _ = sol.solve_loaded(ctx, p)
        t2 = time.perf_counter()
        up.append(t1 - t0)
        so.append(t2 - t1)
        dev.append(res.device_ms / 1e3)
        t0 = time.perf_counter()
        evd.maximise_contrast_bnb(pb, p)
        tot.append(time.perf_counter() - t0)
    m = lambda v: 1e3 * float(np.median(v))
    print(f"cfg {cfg}: upload {m(up):.3f} ms, solve call {m(so):.3f} ms (device {m(dev):.3f}), "
          f"maximise_contrast_bnb {m(tot):.3f} ms")


if __name__ == "__main__":
    main()
