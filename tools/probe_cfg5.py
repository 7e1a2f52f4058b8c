import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import _lib, contrast as con, synth, dist as pdist
from paper_2209_13168_b200.geometry import velocity_domain
b = synth.config_window(5)
ctx = con.load_window(b)
dom = velocity_domain(0.5)
r = np.random.default_rng(0)
for k in (16, 64):
    nus = np.sort(r.uniform(-0.6, -0.2, k))
    lo = np.sort(r.uniform(-0.6, -0.2, 2*k)); hi = lo + 0.003
    con.point_terms(b, nus, ctx=ctx, loaded=True); con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); con.point_terms(b, nus, ctx=ctx, loaded=True); t1 = time.perf_counter()
    con.frontier_terms(b, lo, hi, ctx=ctx, loaded=True); t2 = time.perf_counter()
    print(k, "points %.2f ms" % (1e3*(t1-t0)), "bounds(2k) %.2f ms" % (1e3*(t2-t1)), ctx.frontier_info())
t0 = time.perf_counter(); res = pdist.solve_batched(b, evd.SolverParams(), k=64); print("batched k=64", time.perf_counter()-t0, res)
t0 = time.perf_counter(); res = pdist.solve_batched(b, evd.SolverParams(), k=16); print("batched k=16", time.perf_counter()-t0, res)
t0 = time.perf_counter(); res = pdist.solve_batched(b, evd.SolverParams(), k=8); print("batched k=8", time.perf_counter()-t0, res)
