"""Where the whole-stream pipeline's time goes (tools/bench_stream.py's
50-descent stream): host -> device copy of the raw stream (pageable and
pinned), and the device solve time evd_solve_stream reports.

python tools/probe_stream.py [descents]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import torch
    import paper_2209_13168_b200 as evd
    from bench_stream import make_stream
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    s = make_stream(d)
    params = evd.SolverParams()
    for kind in ("pageable", "pinned"):
        if kind == "pinned":
            x, y, t = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
                       for a in (s.x, s.y, s.t))
            s2 = type(s)(x, y, t, s.polarity, s.geometry)
        else:
            s2 = s
        dev = torch.empty(3 * s.n, dtype=torch.float64, device="cuda")
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i, a in enumerate((s2.x, s2.y, s2.t)):
                dev[i * s.n:(i + 1) * s.n].copy_(torch.from_numpy(a), non_blocking=True)
            torch.cuda.synchronize()
            h2d = time.perf_counter() - t0
        evd.stream_divergence(s2, params)
        t0 = time.perf_counter()
        out = evd.stream_divergence(s2, params)
        tot = time.perf_counter() - t0
        print(f"{kind}: events {s.n} bytes {24 * s.n} h2d {1e3 * h2d:.2f} ms  "
              f"stream_divergence {1e3 * tot:.2f} ms  windows {len(out)}", flush=True)


if __name__ == "__main__":
    main()
