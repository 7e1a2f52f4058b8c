import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2209_13168_b200 import contrast as con, synth
for c in (1, 2, 3):
    b = synth.config_window(c)
    for _ in range(3):
        con.point_terms(b, [-0.4])
