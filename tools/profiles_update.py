"""Copy a tools/round_evidence.sh run (gpurun_out/ev/) into profiles/ with the
ncu summaries the bench line and DESIGN.md cite.

python tools/profiles_update.py [tag]     (tag defaults to r01)
"""

import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EV = os.path.join(ROOT, "gpurun_out", "ev")
PR = os.path.join(ROOT, "profiles")
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_requests_srcunit_tex_op_red.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "launch__shared_mem_per_block_dynamic", "sm__icc_request_hit_rate.pct",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    rep = os.path.join(EV, "k_solve_cfg2.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    h, u, v = rows[0], rows[1], rows[2]
    out = {k: [v[h.index(k)], u[h.index(k)]] for k in WANT if k in h}
    with open(os.path.join(PR, f"ncu_k_solve_cfg2_{tag}.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    to_bytes = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = sum(float(out[k][0]) * to_bytes[out[k][1]]
               for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    with open(os.path.join(PR, "traffic.json"), "w") as fh:
        json.dump({"k_solve_dram_bytes": int(dram),
                   "source": f"ncu --set full, profiles/ncu_k_solve_cfg2_{tag}.json "
                             "(dram__bytes_read.sum + dram__bytes_write.sum)"}, fh, indent=1)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    tmp = os.path.join(EV, "sass.csv")
    with open(tmp, "w") as fh:
        fh.write(src)
    digest = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_profile.py"), tmp],
                            capture_output=True, text=True).stdout
    with open(os.path.join(PR, f"sass_k_solve_cfg2_{tag}.txt"), "w") as fh:
        fh.write(digest)
    for a, b in (("bench.json", f"bench_{tag}_cfg2.json"), ("bench_ref.json", f"bench_ref_{tag}_cfg2.json"),
                 ("launches.csv", f"launches_{tag}_cfg2.csv")):
        shutil.copy(os.path.join(EV, a), os.path.join(PR, b))
    for c in (1, 2, 3):
        shutil.copy(os.path.join(EV, f"trace_cfg{c}.txt"), os.path.join(PR, f"trace_cfg{c}_{tag}.txt"))
    with open(os.path.join(PR, f"probe_events_{tag}.txt"), "w") as fh:
        for c in (2, 3):
            fh.write(open(os.path.join(EV, f"probe_cfg{c}.txt")).read())
    frep = os.path.join(EV, "k_frontier_cfg3.ncu-rep")
    if os.path.exists(frep):
        raw = subprocess.run(["ncu", "-i", frep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout.splitlines()
        rows = list(csv.reader(raw))
        h, u, v = rows[0], rows[1], rows[2]
        fout = {k: [v[h.index(k)], u[h.index(k)]] for k in WANT if k in h}
        with open(os.path.join(PR, f"ncu_k_frontier_cfg3_{tag}.json"), "w") as fh:
            json.dump(fout, fh, indent=1)
    print(json.dumps(out, indent=0)[:800])


if __name__ == "__main__":
    main()
