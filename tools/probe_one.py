"""One evd_probe_events call (for ncu): cfg, width, reps."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2209_13168_b200 import contrast as con, synth
cfg, wd, reps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
b = synth.config_window(cfg)
ctx = con.load_window(b)
out = (ctypes.c_double * reps)()
assert ctx.lib.evd_probe_events(ctx.h, -0.4 - wd / 2, -0.4 + wd / 2, reps, out) == 0
print(np.median(np.array(out[:]) / 1e3))
