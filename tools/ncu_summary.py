"""Summarise one ncu report (the first launch in it) as JSON: the metrics the
bench line and DESIGN.md cite (time, DRAM bytes, issue / occupancy / pipes).

python tools/ncu_summary.py report.ncu-rep out.json
"""

import csv
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_requests_srcunit_tex_op_red.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "launch__shared_mem_per_block_dynamic", "sm__icc_request_hit_rate.pct",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    h, u, v = rows[0], rows[1], rows[2]
    out = {k: [v[h.index(k)], u[h.index(k)]] for k in WANT if k in h}
    out["kernel"] = v[h.index("Kernel Name")] if "Kernel Name" in h else None
    dram = sum(float(out[k][0].replace(",", "")) * TO_BYTES.get(out[k][1], 1)
               for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in out)
    out["dram_bytes"] = int(dram)
    return out


if __name__ == "__main__":
    with open(sys.argv[2], "w") as fh:
        json.dump(summarise(sys.argv[1]), fh, indent=1)
