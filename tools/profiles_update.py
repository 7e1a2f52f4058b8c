"""Copy a tools/round_evidence.sh run (gpurun_out/ev/) into profiles/ with the
ncu summaries the bench line and DESIGN.md cite.

python tools/profiles_update.py [tag]     (tag defaults to r02)
"""

import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
EV = os.path.join(ROOT, "gpurun_out", "ev")
PR = os.path.join(ROOT, "profiles")

from ncu_summary import summarise  # noqa: E402


def digest(rep, out):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    tmp = os.path.join(EV, "sass.csv")
    with open(tmp, "w") as fh:
        fh.write(src)
    d = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_profile.py"), tmp],
                       capture_output=True, text=True).stdout
    with open(out, "w") as fh:
        fh.write(d)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    for rep, name in (("k_solve_cfg2", "k_solve_cfg2"),
                      ("k_frontier_tiles_cfg3", "k_frontier_tiles_cfg3")):
        path = os.path.join(EV, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        with open(os.path.join(PR, f"ncu_{name}_{tag}.json"), "w") as fh:
            json.dump(summarise(path), fh, indent=1)
        digest(path, os.path.join(PR, f"sass_{name}_{tag}.txt"))
    for a, b in (("bench.json", f"bench_{tag}_cfg2.json"), ("bench_ref.json", f"bench_ref_{tag}_cfg2.json"),
                 ("launches.csv", f"launches_{tag}_cfg2.csv"), ("fp64_peak.json", "fp64_peak.json"),
                 ("gpu_tests.log", f"gpu_tests_{tag}.log")):
        if os.path.exists(os.path.join(EV, a)):
            shutil.copy(os.path.join(EV, a), os.path.join(PR, b))
    for c in (1, 2, 3):
        f = os.path.join(EV, f"trace_cfg{c}.txt")
        if os.path.exists(f):
            shutil.copy(f, os.path.join(PR, f"trace_cfg{c}_{tag}.txt"))


if __name__ == "__main__":
    main()
