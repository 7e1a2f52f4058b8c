"""Every device path once, on small windows, for compute-sanitizer
(tools/sanitize.sh runs this under memcheck, racecheck, synccheck and
initcheck).  Each path's result is also checked against the CPU oracle, so a
sanitizer run is a correctness run too.

python tools/sanitize_paths.py
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2209_13168_b200 as evd
    from oracle import oracle as orc
    from paper_2209_13168_b200 import _lib, contrast as con, frontier as fr, synth
    from paper_2209_13168_b200.geometry import velocity_domain

    params = evd.SolverParams()
    r = np.random.default_rng(3)
    small = synth.random_window(r, 64, 48, 1500)
    cfg1 = synth.config_window(1)
    ref_small = orc.maximise_contrast_bnb(small)
    ref_cfg1 = orc.maximise_contrast_bnb(cfg1)

    def same(res, ref):
        return (res.nu, res.contrast, res.iterations) == (ref.nu, ref.contrast, ref.iterations)

    # the solve kernels: speculative 1..4 slots, every CTA size, the filtered path
    for env in ({"EVD_SPEC_K": "1"}, {"EVD_SPEC_K": "2"}, {"EVD_SPEC_K": "4"},
                {"EVD_SPEC_K": "4", "EVD_SOLVE_BLOCK": "384"},
                {"EVD_SPEC_K": "4", "EVD_SOLVE_BLOCK": "768"},
                {"EVD_SPEC_K": "1", "EVD_SOLVE_FILTER": "1"}):
        os.environ.update(env)
        for b, ref in ((small, ref_small), (cfg1, ref_cfg1)):
            res = evd.maximise_contrast_bnb(b, params)
            print("solve", env, b.n, "ok" if same(res, ref) else "MISMATCH", flush=True)
        for k in env:
            del os.environ[k]
    # grouped windows
    wins = [synth.random_window(np.random.default_rng(s), 64, 48, 400 + 37 * s) for s in range(9)]
    samples = evd.estimate_stream_divergence(wins, params)
    ok = all(s.contrast == orc.maximise_contrast_bnb(w).contrast for s, w in zip(samples, wins))
    print("windows", "ok" if ok else "MISMATCH", flush=True)
    # per-call images
    dom = velocity_domain(0.5)
    for lo, hi in ((dom.lo, dom.hi), (-0.5, -0.3), (-0.41, -0.4)):
        _, fi, mk, img = con.bound_terms_many(small, [lo], [hi], images=True)
        oimg, ofi = orc.bound_image(small, lo, hi)
        print("bound", lo, hi, "ok" if np.array_equal(img[0], oimg) and fi[0] == ofi
              else "MISMATCH", flush=True)
    inside, c, imgs = con.point_terms(small, [-0.4, 0.0, -1.9], images=True)
    ok = all(np.array_equal(imgs[j], orc.point_image(small, nu)[0])
             for j, nu in enumerate([-0.4, 0.0, -1.9]))
    print("points", "ok" if ok else "MISMATCH", flush=True)
    # batched frontier: every path, incl. the chunked global path
    ctx = _lib.context()
    lo, hi = fr.uniform_frontier(dom, 6)
    want = con.bound_terms_many(small, lo, hi)
    for path, budget in ((1, None), (2, None), (3, None), (2, 20 * 64 * 48 * 4)):
        ctx.set_option("frontier_path", path)
        if budget:
            ctx.set_option("frontier_image_budget", budget)
        got = con.frontier_terms(small, lo, hi, ctx=ctx)
        ok = all(np.array_equal(a, b) for a, b in zip(got, want[:3]))
        print("frontier path", path, budget, "ok" if ok else "MISMATCH", flush=True)
    ctx.set_option("frontier_path", 0)
    ctx.set_option("frontier_image_budget", 8 << 30)
    # rasterize_segment
    segs = [(0.5, 0.5, 10.25, 7.75), (3.0, 3.0, 3.0, 9.0), (-5.0, 2.5, 70.0, 40.0)]
    got = con.rasterize_segments(segs, evd.SensorGeometry(64, 48), chunk=3)
    ok = all(g == orc.rasterize_segment(s[:2], s[2:], 64, 48) for g, s in zip(got, segs))
    print("raster", "ok" if ok else "MISMATCH", flush=True)
    # EVD1 file -> device decode -> hot pixels -> windows -> solves
    import tempfile
    st = synth.landing_stream(synth.Descent(64, 48, 150, nu=-0.4, duration=1.5, seed=5))
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "s.bin")
        evd.write_event_bin(st, path)
        data = open(path, "rb").read()
    a = evd.stream_divergence_bin(data, params, hot_pixel_k=5.0)
    print("evd1 stream", len(a), "windows", flush=True)
    b = evd.stream_divergence(st, params)
    print("stream", len(b), "windows", flush=True)


if __name__ == "__main__":
    main()
