"""The reference's OWN branch and bound (baseline/_ref/eventdiv/solver.py:79-123,
heapq loop in Python, unmodified) with its per-node functions bound to the
drop-in: eventdiv.contrast / eventdiv.geometry replaced by
paper_2209_13168_b200's, so every contrast_at / bound_terms call is one device
evaluation.  Times one cfg-2 solve with the resident-window cache on and off
and checks the result equals the device-resident solve's.

python tools/ref_loop_bench.py [cfg]   -> one JSON line
"""

import importlib.util
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, ROOT)
sys.path.insert(1, REF)


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import contrast, geometry, synth
    spec = importlib.util.find_spec("eventdiv")
    pkg = importlib.util.module_from_spec(spec)
    sys.modules["eventdiv"] = pkg
    sys.modules["eventdiv.contrast"] = contrast
    sys.modules["eventdiv.geometry"] = geometry
    spec.loader.exec_module(pkg)      # the reference's solver.py binds our contrast functions
    from eventdiv import solver as ref_solver
    assert ref_solver.bound_terms is contrast.bound_terms
    b = synth.config_window(cfg)
    params = ref_solver.SolverParams()
    dev = evd.maximise_contrast_bnb(b, evd.SolverParams())
    out = {"workload": f"cfg{cfg}: reference solver.py loop, per-node calls bound to libevd",
           "events": int(b.n)}
    for cache in (True, False):
        contrast.WINDOW_CACHE = cache
        ref_solver.maximise_contrast_bnb(b, params)  # warm
        t0 = time.perf_counter()
        r = ref_solver.maximise_contrast_bnb(b, params)
        dt = time.perf_counter() - t0
        key = "cached" if cache else "reupload_every_call"
        out[key] = {"seconds_per_solve": dt, "solves_per_s": 1.0 / dt,
                    "device_calls": 2 + 3 * (r.iterations - 1),
                    "identical_to_device_solve": (r.nu, r.contrast, r.iterations) ==
                                                 (dev.nu, dev.contrast, dev.iterations)}
    contrast.WINDOW_CACHE = True
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
