"""Per-iteration device timeline of one evd_solve (globaltimer trace).

python tools/trace_solve.py [cfg] [repeats] [--all] [--spec]
--spec: the speculative-round kernel (k_solve_spec, the default solve), one
row per round (several node evaluations); Mmarks = the round's marks,
"exact%" column replaced by the round's slots.
Per node evaluation (us, from block 0's start of the node):
  b0ev  block 0's events      maxev  the slowest block's events
  bar1  last events -> block 0 leaves barrier 1
  px    block 0's pixels      maxpx  the slowest block's pixels
  bar2  last pixels -> block 0 leaves barrier 2
  step  block 0's BnB step    total  node to node
  Mmarks  segment-image marks of the node (millions)
  G/s     marks per ns of the event phase (the atomic roofline column)
  exact%  events on the exact path
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["EVD_TRACE"] = "1"  # read when the libevd context is created
SPEC = "--spec" in sys.argv
if SPEC:
    os.environ["EVD_TRACE_SPEC"] = "1"
# the probes are compiled only into the diagnostic build
os.environ.setdefault("EVD_LIB", os.path.join(ROOT, "paper_2209_13168_b200", "libevd_trace.so"))

import paper_2209_13168_b200 as evd  # noqa: E402
from paper_2209_13168_b200 import _lib, solver as sol, synth  # noqa: E402

SLOTS = 10


def trace(ctx):
    buf = np.zeros(1 + SLOTS * (1 << 14), dtype=np.int64)
    n = np.zeros(1, dtype=np.int64)
    rc = ctx.lib.evd_solve_trace(ctx.h, _lib.ptr(buf, _lib._i64p), buf.size,
                                 _lib.ptr(n, _lib._i64p))
    assert rc == 0
    return buf[: int(n[0])]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    cfg = int(args[0]) if args else 2
    reps = int(args[1]) if len(args) > 1 else 3
    b = synth.config_window(cfg)
    if os.environ.get("EVD_SHUFFLE"):  # event order does not change any result
        perm = np.random.default_rng(0).permutation(b.n)
        b = type(b)(b.x[perm], b.y[perm], b.t[perm], b.tau, b.geometry)
    for _ in range(reps):
        r, st = sol.solve_window(b, evd.SolverParams())
    tr = trace(_lib.context())
    k = (len(tr) - 1) // SLOTS
    raw = tr[1:1 + SLOTS * k].reshape(k, SLOTS)
    T = raw[:, :8].astype(np.float64) / 1e3
    res, _ = sol.solve_loaded(_lib.context(), evd.SolverParams())
    k = min(k, res.rounds if SPEC else st.point_evals)
    cols = {
        "b0ev": T[:k, 1] - T[:k, 0],
        "maxev": T[:k, 2] - T[:k, 0],
        "bar1": T[:k, 3] - T[:k, 2],
        "px": T[:k, 4] - T[:k, 3],
        "maxpx": T[:k, 5] - T[:k, 3],
        "bar2": T[:k, 6] - T[:k, 5],
        "step": T[:k, 7] - T[:k, 6],
        "total": np.r_[T[1:k, 0] - T[:k - 1, 0], np.nan],
        "Mmarks": raw[:k, 8] / 1e6,
        "G/s": raw[:k, 8] / (T[:k, 2] - T[:k, 0]) / 1e3,  # segment marks / event phase
    }
    if SPEC:
        cols["slots"] = raw[:k, 9].astype(np.float64)
    else:
        cols["exact%"] = 100.0 * raw[:k, 9] / b.n
    print(f"cfg {cfg}: n={b.n} iterations={r.iterations} device_ms={st.device_ms:.3f} "
          f"rounds={res.rounds} "
          f"exact-path share={res.exact_events / (b.n * res.point_evals):.3f}")
    print(("round" if SPEC else "node ") + " ".join(f"{c:>8s}" for c in cols))
    show = range(k) if "--all" in sys.argv else list(range(min(k, 12))) + list(range(max(12, k - 6), k))
    for i in show:
        print(f"{i:4d} " + " ".join(f"{cols[c][i]:8.1f}" for c in cols))
    nar = slice(k // 2, k - 1)
    print("median over the narrow half: " +
          " ".join(f"{c}={np.nanmedian(v[nar]):.1f}" for c, v in cols.items()))
    print("sum: " + " ".join(f"{c}={np.nansum(v):.0f}" for c, v in cols.items()))


if __name__ == "__main__":
    main()


def block_trace(ctx, it_list=(40, 50, 80)):
    S = 20
    blocks = (_lib._i32 * 1)()
    buf = np.zeros(128 * 2048 * S, dtype=np.int64)
    ctx.lib.evd_solve_block_trace(ctx.h, _lib.ptr(buf, _lib._i64p), buf.size, blocks)
    G = blocks[0]
    raw = buf[: 128 * G * S].reshape(128, G, S)
    bt = raw[:, :, :4].astype(np.float64) / 1e3
    for it in it_list:
        t0 = bt[it, 0, 0]
        start = bt[it, :, 0] - t0
        ev = bt[it, :, 1] - bt[it, :, 0]
        px = bt[it, :, 2] - bt[it, :, 1]
        step = bt[it, :, 3] - bt[it, :, 2]
        print(f"node {it}: start skew p50/max {np.median(start):.1f}/{start.max():.1f} us; "
              f"events p50/p90/max {np.median(ev):.1f}/{np.percentile(ev, 90):.1f}/{ev.max():.1f} "
              f"(argmax block {int(ev.argmax())}); px+bar1 p50/max {np.median(px):.1f}/{px.max():.1f}; "
              f"step+bar2 p50/max {np.median(step):.1f}/{step.max():.1f}")
        c = raw[it, :, 4:13].astype(np.float64)
        names = ["mu/acc", "cuts", "A/B px", "blkadd", "->bar2", "stage", "top", "bnb"]
        d = np.diff(c, axis=1)
        med = np.median(d, axis=0)
        print("   block cycles (median over blocks): " +
              " ".join(f"{n}={v:.0f}" for n, v in zip(names, med)))
        e = raw[it, :, 13:16].astype(np.float64)
        pre = e[:, 0] - raw[it, :, 5]
        print("   cut detail: mu=%.0f leaves=%.0f sync=%.0f" % (
            np.median(pre), np.median(e[:, 1] - e[:, 0]), np.median(e[:, 2] - e[:, 1])))
        f = raw[it, :, 16:20].astype(np.float64)
        print("   eval_cut entry after mu: %.0f cycles" % np.median(f[:, 3] - e[:, 0]))
        print("   leaf detail (thread 0): cut_leaf0=%.0f leaves[]=%.0f leaf8=%.0f rest=%.0f" % (
            np.median(f[:, 0] - e[:, 0]), np.median(f[:, 1] - f[:, 0]),
            np.median(f[:, 2] - f[:, 1]), np.median(e[:, 1] - f[:, 2])))


if "--blocks" in sys.argv:
    its = [int(x) for a in sys.argv if a.startswith("--nodes=") for x in a.split("=")[1].split(",")]
    block_trace(_lib.context(), *([its] if its else []))
