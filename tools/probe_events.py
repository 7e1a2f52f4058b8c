"""Device time of the solve kernel's exact event pass (evd_probe_events) for
child evaluations of decreasing width around the optimum.

python tools/probe_events.py [cfg] [reps]   -> one line per width
"""

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2209_13168_b200 import _lib, contrast as con, synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    b = synth.config_window(cfg)
    if os.environ.get("EVD_SHUFFLE"):  # event order does not change any result
        perm = np.random.default_rng(0).permutation(b.n)
        b = type(b)(b.x[perm], b.y[perm], b.t[perm], b.tau, b.geometry)
    ctx = con.load_window(b)
    out = (ctypes.c_double * reps)()
    parts = []
    for w in (1.0, 1e-1, 1e-2, 1e-3, 1e-4, 1e-5):
        lo, hi = -0.4 - w / 2, -0.4 + w / 2
        rc = ctx.lib.evd_probe_events(ctx.h, lo, hi, reps, out)
        assert rc == 0, ctx.error_text()
        us = np.array(out[:]) / 1e3
        parts.append(f"w={w:g}: {np.median(us[1:]):.1f}")
    print(f"cfg {cfg} n={b.n} event pass us (median of {reps - 1}): " + "  ".join(parts))


if __name__ == "__main__":
    main()
