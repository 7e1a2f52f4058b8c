"""Batched bound evaluation at small K: the frontier kernels (lane = interval)
against per-interval k_bound_image launches (lane = event), cfg 5 window.

python tools/probe_small_k.py [cfg]
"""
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
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    b = synth.config_window(cfg)
    ctx = con.load_window(b)
    dom = velocity_domain(b.tau)
    for depth in (0, 1, 2, 3, 4, 5):
        lo, hi = fr.uniform_frontier(dom, depth)
        out = {}
        for name, fn in (("tiles", lambda: con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)),
                         ("per_interval", lambda: con.bound_terms_many(b, lo, hi, ctx=ctx,
                                                                       loaded=True))):
            if name == "tiles":
                ctx.set_option("frontier_path", 1)
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            out[name] = (time.perf_counter() - t0, r)
            ctx.set_option("frontier_path", 0)
        same = all(np.array_equal(u, v) for u, v in zip(out["tiles"][1], out["per_interval"][1][:3]))
        print(f"K={lo.size}: tiles {1e3 * out['tiles'][0]:.2f} ms, per-interval "
              f"{1e3 * out['per_interval'][0]:.2f} ms, same={same}", flush=True)


if __name__ == "__main__":
    main()
