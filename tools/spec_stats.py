"""Node evaluations per solve with and without speculative rounds.

python tools/spec_stats.py [cfg ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import _lib, solver as sol, synth
    from paper_2209_13168_b200.contrast import load_window
    for c in [int(x) for x in sys.argv[1:]] or [1, 2, 3]:
        b = synth.config_window(c)
        ctx = load_window(b)
        res, _ = sol.solve_loaded(ctx, evd.SolverParams())
        res, _ = sol.solve_loaded(ctx, evd.SolverParams())
        print(f"cfg {c}: iterations={res.iterations} point_evals={res.point_evals} "
              f"evaluations={res.exact_events / b.n:.1f} device_ms={res.device_ms:.3f} "
              f"max_frontier={res.max_frontier}", flush=True)


if __name__ == "__main__":
    main()
