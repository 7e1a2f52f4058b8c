"""Config 5 (1280x720, 5,327,641 events): the reference-order device solve and
the batched-frontier solve (k nodes per round; the rounds' evaluations are what
a multi-GPU run splits over ranks).

python tools/bench_cfg5.py [k ...]   -> JSON lines
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# reference maximise_contrast_bnb on this window
REF = {"nu": -0.4000001722040176, "contrast": 753.9103765755924,
       "bound_gap": 0.015945095486131322, "iterations": 144, "cpu_s": 1791.5}


def main():
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import dist as pdist, solver as sol, synth

    ks = [int(a) for a in sys.argv[1:]] or [32, 128]
    b = synth.config_window(5)
    params = evd.SolverParams()
    sol.solve_window(b, params)  # warm
    r, st = sol.solve_window(b, params)
    same = (r.nu, r.contrast, r.bound_gap, r.iterations) == (
        REF["nu"], REF["contrast"], REF["bound_gap"], REF["iterations"])
    print(json.dumps({"workload": f"cfg5 exact solve: 1280x720, {b.n} events",
                      "device_s": st.device_ms / 1e3, "iterations": r.iterations,
                      "bound_evals": st.bound_evals, "marks": None,
                      "identical_to_reference": same, "reference_cpu_s": REF["cpu_s"],
                      "nu": r.nu, "contrast": r.contrast}), flush=True)
    for k in ks:
        t0 = time.perf_counter()
        res = pdist.solve_batched(b, params, k=k)
        dt = time.perf_counter() - t0
        print(json.dumps({"workload": f"cfg5 batched frontier k={k}", "wall_s": dt,
                          "rounds": res.rounds, "nodes": res.nodes,
                          "bound_evals": res.bound_evals, "contrast": res.contrast,
                          "nu": res.nu, "within_gamma_of_reference":
                              res.contrast >= REF["contrast"] - params.gamma,
                          "divergence": pdist.divergence_of(res, b.tau)}), flush=True)


if __name__ == "__main__":
    main()
