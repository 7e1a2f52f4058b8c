"""Launch the standalone point / bound kernels over a range of interval widths
(run under `ncu --metrics gpu__time_duration.sum` to get per-launch times).

python tools/probe_kernels.py [cfg]
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2209_13168_b200 import contrast as con, synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
b = synth.config_window(cfg)
ivs = [(-1.999998, 0.0), (-0.5, -0.25), (-0.41, -0.39), (-0.4001, -0.3999), (-0.40001, -0.39999),
       (-1e-4, 0.0), (-1.5, -1.4999)]
s, fi, marks, _ = con.bound_terms_many(b, [a for a, _ in ivs], [c for _, c in ivs])
for (lo, hi), m in zip(ivs, marks):
    print(f"bound [{lo}, {hi}] marks={int(m)} per event {int(m) / b.n:.2f}")
nus = [-0.4, 0.0, -1.0, -1.9]
ins, c, _ = con.point_terms(b, nus)
print("points", list(zip(nus, ins.tolist())))
