"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the development container only (needs /root/reference, numba):

    python tests/golden/make_golden.py [--big]

It imports ``eventdiv`` from /root/reference/pkg/src with bytecode and numba
caches redirected away from the (read-only) reference tree, and writes small
``.npz`` / ``.json`` fixtures next to this script.  The fixtures are committed;
nothing on the GPU box reads /root/reference.

Fixtures:
  segments.npz  rasterize_segment pixel sets (contrast.py:206-222) for random
                and adversarial segments on several grids
  images.npz    accumulate_image / image_contrast / upper_bound_image /
                _bound_image_kernel / bound_terms outputs for small batches
  bnb.json      maximise_contrast_bnb results (+ per-node trace for a few
                batches) and grid_search_oracle results
  synth.json    checksums of the reference simulator's windows for the
                SURVEY §8(d) configurations (pins paper_2209_13168_b200.synth)
  preproc.npz   pixel_counts / remove_hot_pixels / rescale_events (events.py:273-313)
                outputs on test-suite streams, landing streams with injected hot
                pixels, and rescale targets
  nonfinite.npz / .json  point / bound images and BnB results for windows
                with NaN, infinite and huge coordinates and NaN timestamps
  evd1.npz      EVD1 files (parse_event_bin, events.py:186-206): valid bodies
                (sorted, unsorted with equal timestamps, large t_us) with the
                reference's decoded arrays, and malformed / invalid bodies
                with the reference's exception class and message
"""

from __future__ import annotations

import hashlib
import heapq
import itertools
import json
import os
import sys

sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/evd_numba_cache")
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))

import numpy as np  # noqa: E402
from eventdiv import contrast as con  # noqa: E402
from eventdiv import solver as sol  # noqa: E402
from eventdiv.events import EventBatch, SensorGeometry, batch_stream  # noqa: E402
from eventdiv.geometry import VelocityInterval, velocity_domain, warp_batch  # noqa: E402
from eventdiv.simulator import SimConfig, generate_landing_events  # noqa: E402


def bits(v: float) -> str:
    return np.float64(v).tobytes().hex()


# ------------------------------------------------------------------ segments
def adversarial_segments(rng, w, h, n_random):
    segs = []
    for _ in range(n_random):
        segs.append(rng.uniform(-4, max(w, h) + 4, 4))
    for _ in range(n_random // 4):  # integer corners, diagonals through lattice points
        segs.append(rng.integers(-2, max(w, h) + 3, 4).astype(float))
    for _ in range(n_random // 4):  # axis-aligned, on and off grid lines
        a = rng.uniform(-2, w + 2)
        b, c = rng.uniform(-2, h + 2, 2)
        if rng.random() < 0.5:
            a = float(np.round(a))
        segs.append(np.array([a, b, a, c]) if rng.random() < 0.5 else np.array([b, a, c, a]))
    for _ in range(n_random // 8):  # lattice diagonals k*(1,1), k*(1,-1), k*(2,1)
        x0, y0 = rng.integers(-1, w + 1), rng.integers(-1, h + 1)
        dx, dy = [(1, 1), (1, -1), (2, 1), (1, 2), (-3, 1)][rng.integers(0, 5)]
        k = rng.integers(1, 8)
        segs.append(np.array([x0, y0, x0 + k * dx, y0 + k * dy], dtype=float))
    for _ in range(n_random // 8):  # very long, radial through the image
        ang = rng.uniform(0, 2 * np.pi)
        r0, r1 = rng.uniform(0, 5), 10.0 ** rng.uniform(2, 8)
        cx, cy = w / 2, h / 2
        segs.append(np.array([cx + r0 * np.cos(ang), cy + r0 * np.sin(ang),
                              cx + r1 * np.cos(ang), cy + r1 * np.sin(ang)]))
    for _ in range(n_random // 8):  # tiny and degenerate
        p = rng.uniform(-1, max(w, h) + 1, 2)
        if rng.random() < 0.3:
            p = np.round(p)
        q = p + rng.normal(0, 1e-6, 2) if rng.random() < 0.6 else p.copy()
        segs.append(np.concatenate([p, q]))
    return [np.asarray(s, dtype=np.float64) for s in segs]


def make_segments():
    rng = np.random.default_rng(20260101)
    all_segs, dims, offs, pix = [], [], [0], []
    for (w, h, n) in [(8, 8, 200), (16, 16, 800), (32, 32, 1600), (64, 48, 800), (7, 5, 200)]:
        g = SensorGeometry(w, h)
        for s in adversarial_segments(rng, w, h, n):
            cells = sorted(con.rasterize_segment((s[0], s[1]), (s[2], s[3]), g))
            all_segs.append(s)
            dims.append((w, h))
            pix.extend(cells)
            offs.append(len(pix))
    np.savez_compressed(os.path.join(HERE, "segments.npz"),
                        segs=np.array(all_segs), dims=np.array(dims, dtype=np.int32),
                        offsets=np.array(offs, dtype=np.int64),
                        pixels=np.array(pix, dtype=np.int32).reshape(-1, 2))
    print("segments:", len(all_segs), "pixels:", len(pix))


# ------------------------------------------------------------------ images
def sim_windows(nu, duration, seed, n_points, w, h, tau=0.5):
    cfg = SimConfig(z0=1.0, nu=nu, geometry=SensorGeometry(w, h), duration=duration,
                    n_points=n_points, seed=seed)
    stream, _ = generate_landing_events(cfg)
    return [b for b in batch_stream(stream, tau) if b.n]


def image_cases():
    rng = np.random.default_rng(12345)
    cases = []

    def rand_batch(w, h, n, tau=0.5):
        x = rng.uniform(0, w, n)
        y = rng.uniform(0, h, n)
        t = np.sort(rng.uniform(0, tau, n))
        return EventBatch(x, y, t, tau, SensorGeometry(w, h))

    cases.append(("random64", rand_batch(64, 64, 300)))
    cases.append(("random32", rand_batch(32, 32, 200)))
    cases.append(("random_rect", rand_batch(37, 23, 900, tau=0.7)))
    cases.append(("sim64", sim_windows(-0.4, 1.5, 3, 400, 64, 64)[0]))
    cases.append(("sim64_w2", sim_windows(-0.4, 1.5, 3, 400, 64, 64)[2]))
    cases.append(("sim160", sim_windows(-0.3, 2.5, 0, 600, 160, 90)[1]))
    # special events: FOE, integer coordinates, t = tau, t = 0, pixel corners
    g = SensorGeometry(40, 30)
    xs = [20.0, 20.0, 0.0, 39.999, 10.0, 10.5, 31.0, 5.0, 20.0, 0.25]
    ys = [15.0, 3.0, 0.0, 29.999, 10.0, 10.5, 7.0, 25.0, 29.0, 14.0]
    ts = [0.1, 0.5, 0.0, 0.25, 0.5, 0.0, 0.2, 0.49, 0.0, 0.3]
    order = np.argsort(ts, kind="stable")
    cases.append(("special", EventBatch(np.array(xs)[order], np.array(ys)[order],
                                        np.array(ts)[order], 0.5, g)))
    return cases


def intervals_for(batch, rng):
    lo0, hi0 = velocity_domain(batch.tau).lo, velocity_domain(batch.tau).hi
    ivs = [(lo0, hi0)]
    a = VelocityInterval(lo0, hi0)
    for _ in range(6):  # left-most descent (near-singular warps)
        a = a.split()[0]
        ivs.append((a.lo, a.hi))
    b = VelocityInterval(lo0, hi0)
    for _ in range(12):  # descent towards nu = -0.4
        l, r = b.split()
        b = l if l.lo <= -0.4 <= l.hi else r
        ivs.append((b.lo, b.hi))
    for _ in range(8):
        lo, hi = np.sort(rng.uniform(lo0, hi0, 2))
        ivs.append((float(lo), float(hi)))
    nu = float(rng.uniform(lo0, hi0))
    ivs.append((nu, nu))  # singleton
    ivs.append((-0.4, -0.4))
    return ivs


def make_images():
    rng = np.random.default_rng(777)
    out = {}
    meta = []
    for name, batch in image_cases():
        g = batch.geometry
        out[f"{name}/x"], out[f"{name}/y"], out[f"{name}/t"] = batch.x, batch.y, batch.t
        lo0 = velocity_domain(batch.tau).lo
        nus = [0.0, -0.4, lo0, 0.5 * lo0, float(rng.uniform(lo0, 0)), -1e-300]
        pts = []
        for j, nu in enumerate(nus):
            img = con.accumulate_image(batch, nu)
            out[f"{name}/point{j}"] = img.counts.astype(np.uint32)
            pts.append({"nu": bits(nu), "in_image": img.in_image_events,
                        "contrast": bits(con.image_contrast(img)),
                        "contrast_expanded": bits(con.image_contrast_expanded(img))})
        bnds = []
        for j, (lo, hi) in enumerate(intervals_for(batch, rng)):
            iv = VelocityInterval(lo, hi)
            ub = con.upper_bound_image(batch, iv)
            x0, y0 = warp_batch(batch, lo)
            x1, y1 = warp_batch(batch, hi)
            counts = np.zeros((g.height, g.width))
            stamp = np.full((g.height, g.width), -1, dtype=np.int64)
            fi = con._bound_image_kernel(x0, y0, x1, y1, g.width, g.height, counts, stamp)
            assert np.array_equal(counts, ub.counts)
            bt = con.bound_terms(batch, iv)
            out[f"{name}/bound{j}"] = ub.counts.astype(np.uint32)
            bnds.append({"lo": bits(lo), "hi": bits(hi), "marks": ub.in_image_events,
                         "fully_inside": int(fi), "s_bar": bits(bt.s_bar),
                         "mu_lower": bits(bt.mu_lower), "c_bar": bits(bt.c_bar)})
        meta.append({"name": name, "width": g.width, "height": g.height, "tau": bits(batch.tau),
                     "n": batch.n, "points": pts, "bounds": bnds})
    np.savez_compressed(os.path.join(HERE, "images.npz"), **out)
    with open(os.path.join(HERE, "images.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("images:", len(meta), "cases")


# ------------------------------------------------------------------ bnb
def traced_bnb(batch, params):
    """The reference loop (solver.py:79-123) driven through the reference's own
    contrast_at / bound_terms, recording every node; asserts it reproduces
    maximise_contrast_bnb exactly."""
    dom = velocity_domain(batch.tau, params.epsilon)
    nu_hat = dom.center
    c_hat = sol.contrast_at(batch, nu_hat)
    ctr = itertools.count()
    rb = con.bound_terms(batch, dom)
    trace = [{"kind": "root", "lo": bits(dom.lo), "hi": bits(dom.hi), "c_bar": bits(rb.c_bar),
              "s_bar": bits(rb.s_bar), "mu_lower": bits(rb.mu_lower), "c_center": bits(c_hat)}]
    heap = [(-rb.c_bar, next(ctr), dom)]
    it = 0
    gapv = 0.0
    while heap:
        neg, _, iv = heapq.heappop(heap)
        it += 1
        gap = -neg - c_hat
        if gap <= params.gamma or iv.width < params.min_interval_width:
            gapv = max(gap, 0.0)
            break
        c = iv.center
        cc = sol.contrast_at(batch, c)
        node = {"kind": "node", "lo": bits(iv.lo), "hi": bits(iv.hi), "c_center": bits(cc)}
        if cc >= c_hat:
            nu_hat, c_hat = c, cc
        kids = []
        for ch in iv.split():
            b = con.bound_terms(batch, ch)
            kids.append({"c_bar": bits(b.c_bar), "s_bar": bits(b.s_bar),
                         "mu_lower": bits(b.mu_lower)})
            if b.c_bar >= c_hat:
                heapq.heappush(heap, (-b.c_bar, next(ctr), ch))
        node["children"] = kids
        trace.append(node)
    ref = sol.maximise_contrast_bnb(batch, params)
    assert (ref.nu, ref.contrast, ref.bound_gap, ref.iterations) == (nu_hat, c_hat, gapv, it)
    return ref, trace


def res_dict(r):
    return {"nu": bits(r.nu), "contrast": bits(r.contrast), "bound_gap": bits(r.bound_gap),
            "iterations": r.iterations, "runtime_s": r.runtime}


def make_bnb(big: bool):
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2209_13168_b200 import synth
    params = sol.SolverParams()
    out = {"small": [], "configs": {}, "grid": [], "sequence": []}
    rng = np.random.default_rng(4242)
    windows = sim_windows(-0.4, 1.5, 3, 400, 64, 64)
    windows += sim_windows(-0.3, 2.5, 0, 600, 160, 90)[:3]
    windows += [EventBatch(rng.uniform(0, 64, 500), rng.uniform(0, 64, 500),
                           np.sort(rng.uniform(0, 0.5, 500)), 0.5, SensorGeometry(64, 64))]
    windows += [EventBatch(np.array([32.0]), np.array([32.0]), np.array([0.1]), 0.5,
                           SensorGeometry(64, 64))]
    arrays = {}
    for j, b in enumerate(windows):
        r, trace = traced_bnb(b, params)
        arrays[f"w{j}/x"], arrays[f"w{j}/y"], arrays[f"w{j}/t"] = b.x, b.y, b.t
        out["small"].append({"width": b.geometry.width, "height": b.geometry.height,
                             "tau": bits(b.tau), "t_start": bits(b.t_start), "n": b.n,
                             "result": res_dict(r), "trace": trace})
        if j < 3:
            for npts in (2, 64, 512):
                nu, c = sol.grid_search_oracle(b, params, npts)
                out["grid"].append({"window": j, "n_points": npts, "nu": bits(nu), "c": bits(c)})
    # iteration cap on window 0
    try:
        sol.maximise_contrast_bnb(windows[0], sol.SolverParams(max_iterations=2))
    except sol.IterationLimitError as e:
        out["iteration_limit"] = {"window": 0, "max_iterations": 2, "nu": bits(e.nu),
                                  "contrast": bits(e.contrast), "iterations": e.iterations}
    np.savez_compressed(os.path.join(HERE, "bnb_windows.npz"), **arrays)
    cfgs = [1, 2] + ([3] if big else [])
    for cfg in cfgs:
        b = synth.config_window(cfg)
        r, trace = traced_bnb(b, params)
        out["configs"][str(cfg)] = {"n": b.n, "result": res_dict(r), "trace": trace}
        print("cfg", cfg, b.n, r)
    for k in (0, 1, 2, 3, 1000, 1999):
        b = synth.sequence_window(k)
        r = sol.maximise_contrast_bnb(b, params)
        out["sequence"].append({"k": k, "n": b.n, "result": res_dict(r)})
    with open(os.path.join(HERE, "bnb.json"), "w") as fh:
        json.dump(out, fh, indent=1)


# ------------------------------------------------------------------ evd1
def make_evd1():
    import struct
    from eventdiv import events as ev
    rng = np.random.default_rng(777)
    rec = np.dtype([("t_us", "<u8"), ("x", "<f4"), ("y", "<f4"), ("p", "i1")])

    def body(w, h, t_us, x, y, p, count=None):
        r = np.empty(len(t_us), dtype=rec)
        r["t_us"], r["x"], r["y"], r["p"] = t_us, x, y, p
        n = len(t_us) if count is None else count
        return struct.pack("<4sIIQ", b"EVD1", w, h, n) + r.tobytes()

    cases = {}
    n = 5000
    t = np.sort(rng.integers(0, 3 * 10**6, n)).astype(np.uint64)
    xs, ys = rng.uniform(0, 64, n), rng.uniform(0, 48, n)
    ps = rng.choice([-1, 1], n).astype(np.int8)
    cases["sorted"] = body(64, 48, t, xs, ys, ps)
    tu = rng.integers(0, 2000, n).astype(np.uint64) * 1000  # many equal timestamps
    cases["unsorted_ties"] = body(64, 48, tu, xs, ys, ps)
    big = (np.uint64(2**60) + rng.integers(0, 2**40, 64).astype(np.uint64))
    cases["large_t"] = body(64, 48, big, xs[:64], ys[:64], ps[:64])
    cases["empty"] = body(8, 8, np.empty(0, np.uint64), [], [], [])
    cases["edge_coords"] = body(4, 4, np.arange(4, dtype=np.uint64),
                                np.array([0.0, 3.9999998, 0.0, 3.5], np.float32),
                                np.array([0.0, 3.9999998, 3.9999998, 0.0], np.float32),
                                np.array([1, -1, 1, -1], np.int8))
    bad = {
        "short_header": b"EVD1\0\0",
        "bad_magic": b"NOPE" + b"\0" * 16,
        "truncated": body(4, 4, np.arange(3, dtype=np.uint64), [1.0] * 3, [1.0] * 3, [1] * 3,
                          count=5),
        "out_of_frame": body(4, 4, np.arange(3, dtype=np.uint64), [1.0, 4.0, 1.0], [1.0] * 3,
                             [1] * 3),
        "negative_coord": body(4, 4, np.arange(2, dtype=np.uint64), [1.0, -0.5], [1.0] * 2,
                               [1] * 2),
        "nan_coord": body(4, 4, np.arange(2, dtype=np.uint64), [1.0, np.nan], [1.0] * 2, [1] * 2),
        "bad_polarity": body(4, 4, np.arange(2, dtype=np.uint64), [1.0] * 2, [1.0] * 2, [1, 0]),
        "zero_width": body(0, 4, np.arange(1, dtype=np.uint64), [0.0], [0.0], [1]),
    }
    out, meta = {}, {"valid": [], "invalid": {}}
    for name, data in cases.items():
        st = ev.parse_event_bin(data)
        out[f"{name}_data"] = np.frombuffer(data, np.uint8)
        for k in ("x", "y", "t"):
            out[f"{name}_{k}"] = getattr(st, k)
        out[f"{name}_p"] = st.polarity
        out[f"{name}_geom"] = np.array([st.geometry.width, st.geometry.height])
        meta["valid"].append(name)
    for name, data in bad.items():
        out[f"bad_{name}_data"] = np.frombuffer(data, np.uint8)
        try:
            ev.parse_event_bin(data)
            meta["invalid"][name] = None
        except Exception as exc:  # the reference's class and message
            meta["invalid"][name] = [type(exc).__name__, str(exc)]
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "evd1.npz"), **out)


# ------------------------------------------------------------------ preprocessing
def make_preproc():
    from eventdiv import events as ev
    rng = np.random.default_rng(4242)
    cases = []

    def stream(x, y, t, w, h, p=None):
        x = np.asarray(x, np.float64)
        p = np.ones(len(x), np.int8) if p is None else np.asarray(p, np.int8)
        return ev.EventStream(x, np.asarray(y, np.float64), np.asarray(t, np.float64), p,
                              SensorGeometry(w, h))

    xs, ys = np.meshgrid(np.arange(3) + 0.5, np.arange(3) + 0.5)
    cases.append(("uniform", stream(xs.ravel(), ys.ravel(), np.arange(9) * 0.01, 8, 8), 5.0))
    hx, hy, ht, t0 = [], [], [], 0.0
    for i in range(8):
        hx.append(i + 0.5); hy.append(0.5); ht.append(t0); t0 += 1e-4
    for i in range(8):
        for _ in range(2):
            hx.append(i + 0.5); hy.append(1.5); ht.append(t0); t0 += 1e-4
    for _ in range(1000):
        hx.append(7.5); hy.append(7.5); ht.append(t0); t0 += 1e-4
    cases.append(("hot", stream(hx, hy, ht, 8, 8), 5.0))
    n = 2000
    cases.append(("random8", stream(rng.uniform(0, 8, n), rng.uniform(0, 8, n),
                                    np.sort(rng.uniform(0, 1, n)), 8, 8,
                                    rng.choice([-1, 1], n)), 10.0))
    stream_l, _ = generate_landing_events(SimConfig(
        z0=1.0, nu=-0.3, geometry=SensorGeometry(64, 48), duration=1.5, n_points=400,
        event_spacing_px=1.0, seed=9))
    # inject hot pixels: many events on a few pixels, merged in time order
    inj_t = np.sort(rng.uniform(0, 1.5, 3000))
    inj_x = rng.choice([3.5, 40.25, 63.75], 3000)
    inj_y = rng.choice([1.5, 20.5, 47.5], 3000)
    allx = np.concatenate([stream_l.x, inj_x]); ally = np.concatenate([stream_l.y, inj_y])
    allt = np.concatenate([stream_l.t, inj_t]); allp = np.concatenate([stream_l.polarity,
                                                                       np.ones(3000, np.int8)])
    order = np.argsort(allt, kind="stable")
    landing = stream(allx[order], ally[order], allt[order], 64, 48, allp[order])
    cases.append(("landing_hot10", landing, 10.0))
    cases.append(("landing_hot3", landing, 3.0))
    cases.append(("landing_clean", stream_l, 10.0))
    n = 20000  # dense: median and MAD well above 1, an even count of nonzero pixels
    dx = np.concatenate([rng.uniform(0, 16, n), np.full(900, 2.5), np.full(700, 13.75)])
    dy = np.concatenate([rng.uniform(0, 12, n), np.full(900, 7.5), np.full(700, 0.25)])
    dt = np.sort(rng.uniform(0, 2, len(dx)))
    perm = rng.permutation(len(dx))
    dense = stream(dx[perm], dy[perm], dt, 16, 12, rng.choice([-1, 1], len(dx)))
    cases.append(("dense4", dense, 4.0))
    cases.append(("dense2_5", dense, 2.5))
    out, meta = {}, {"hot": [], "rescale": []}
    for name, st, k in cases:
        kept = ev.remove_hot_pixels(st, k=k)
        counts = ev.pixel_counts(st)
        nz = counts[counts > 0].astype(np.float64)
        med = np.median(nz); mad = np.median(np.abs(nz - med))
        for key, arr in (("x", st.x), ("y", st.y), ("t", st.t), ("p", st.polarity),
                         ("kx", kept.x), ("ky", kept.y), ("kt", kept.t), ("kp", kept.polarity),
                         ("counts", counts)):
            out[f"{name}_{key}"] = arr
        meta["hot"].append({"name": name, "w": st.geometry.width, "h": st.geometry.height,
                            "k": k, "threshold": bits(float(med + k * mad))})
    for name, st, (w2, h2) in (("land_half", stream_l, (32, 24)), ("land_odd", stream_l, (97, 61)),
                               ("example", stream([640.0], [380.0], [0.0], 1280, 760), (160, 90))):
        r = ev.rescale_events(st, SensorGeometry(w2, h2))
        for key, arr in (("x", st.x), ("y", st.y), ("t", st.t), ("p", st.polarity),
                         ("rx", r.x), ("ry", r.y)):
            out[f"{name}_{key}"] = arr
        meta["rescale"].append({"name": name, "w": st.geometry.width, "h": st.geometry.height,
                                "w2": w2, "h2": h2})
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "preproc.npz"), **out)


# ------------------------------------------------------------------ synth
def make_synth():
    out = {}
    for cfg, (w, h, npts, sp) in {1: (240, 180, 1450, 1.0), 2: (346, 260, 10000, 1.0),
                                  3: (640, 480, 13000, 0.5), 5: (1280, 720, 38000, 0.5)}.items():
        stream, _ = generate_landing_events(SimConfig(
            z0=1.0, nu=-0.4, geometry=SensorGeometry(w, h), duration=2.0, n_points=npts,
            event_spacing_px=sp, seed=0))
        b = batch_stream(stream, 0.5)[0]
        hsh = hashlib.sha256(b.x.tobytes() + b.y.tobytes() + b.t.tobytes()).hexdigest()
        out[str(cfg)] = {"n": b.n, "sha256": hsh, "stream_n": stream.n}
    with open(os.path.join(HERE, "synth.json"), "w") as fh:
        json.dump(out, fh, indent=1)


# ------------------------------------------------------------------ cfg-3 frontier
def _frontier_leaf(args):
    """bound_terms (contrast.py:241-251) of one leaf, run by the reference's own
    numba kernel; also the mark total (upper_bound_image().in_image_events)."""
    j, lo, hi = args
    from eventdiv.geometry import VelocityInterval
    b = _FRONTIER_BATCH
    g = b.geometry
    x0, y0, x1, y1 = con._segment_endpoints(b, VelocityInterval(lo, hi))
    counts = np.zeros((g.height, g.width), dtype=np.float64)
    stamp = np.full((g.height, g.width), -1, dtype=np.int64)
    fi = con._bound_image_kernel(x0, y0, x1, y1, g.width, g.height, counts, stamp)
    bound = con.bound_terms(b, VelocityInterval(lo, hi)) if j % 512 == 0 else None
    s_bar = float(np.sum(counts**2))
    if bound is not None:  # the public entry point agrees with the kernel call above
        assert bound.s_bar == s_bar and bound.mu_lower == fi / g.n_pixels
    return j, s_bar, int(fi), float(counts.sum())


_FRONTIER_BATCH = None


def make_frontier(procs: int = 8):
    """The SURVEY §8(d) cfg-3 frontier: all 4096 depth-12 leaves of the root
    bisection of the 640x480, 999,557-event window, each bound evaluated by the
    reference (one numba _bound_image_kernel per leaf, leaves spread over
    `procs` worker processes).  The window is the reference simulator's own."""
    global _FRONTIER_BATCH
    import multiprocessing as mp
    from eventdiv.geometry import velocity_domain
    stream, _ = generate_landing_events(SimConfig(
        z0=1.0, nu=-0.4, geometry=SensorGeometry(640, 480), duration=2.0, n_points=13000,
        event_spacing_px=0.5, seed=0))
    _FRONTIER_BATCH = batch_stream(stream, 0.5)[0]
    level = [velocity_domain(0.5)]
    for _ in range(12):
        level = [c for iv in level for c in iv.split()]
    jobs = [(j, iv.lo, iv.hi) for j, iv in enumerate(level)]
    with mp.get_context("fork").Pool(procs) as pool:
        rows = sorted(pool.map(_frontier_leaf, jobs, chunksize=16))
    s_bar = np.array([r[1] for r in rows], dtype=np.float64)
    fi = np.array([r[2] for r in rows], dtype=np.int64)
    marks = np.array([r[3] for r in rows], dtype=np.float64)
    assert np.all(s_bar < 2.0**53) and np.all(marks < 2.0**53)  # exact integers
    hsh = hashlib.sha256(_FRONTIER_BATCH.x.tobytes() + _FRONTIER_BATCH.y.tobytes() +
                         _FRONTIER_BATCH.t.tobytes()).hexdigest()
    np.savez_compressed(os.path.join(HERE, "frontier_cfg3.npz"),
                        lo=np.array([r[1] for r in jobs]), hi=np.array([r[2] for r in jobs]),
                        s_bar=s_bar.astype(np.uint64), fully_inside=fi,
                        marks=marks.astype(np.uint64),
                        window_sha256=np.frombuffer(hsh.encode(), np.uint8))
    print("frontier: 4096 leaves, marks", int(marks.sum()))


def make_nonfinite():
    """Windows with NaN / infinite / huge coordinates and NaN timestamps (the
    reference's EventBatch validates only the t range, so these reach the
    path): point images, bound images and the BnB result."""
    import warnings
    rng = np.random.default_rng(4711)
    out, meta = {}, []
    w, h, n = 40, 30, 600
    for case in range(4):
        x = rng.uniform(0, w, n)
        y = rng.uniform(0, h, n)
        t = np.sort(rng.uniform(0, 0.5, n))
        k = rng.choice(n, 40, replace=False)
        if case == 0:
            x[k[:20]] = np.nan
            y[k[20:]] = np.nan
        elif case == 1:
            t[k] = np.nan
        elif case == 2:
            x[k[:20]] = np.inf
            y[k[20:]] = -np.inf
        else:
            x[k[:20]] = 1e308
            x[k[20:]] = -1e308
        b = EventBatch(x, y, t, 0.5, SensorGeometry(w, h))
        name = f"nf{case}"
        out[f"{name}/x"], out[f"{name}/y"], out[f"{name}/t"] = x, y, t
        lo0 = velocity_domain(0.5).lo
        ivs = [(lo0, 0.0), (-0.5, -0.3), (-0.41, -0.4)]
        rec = {"name": name, "width": w, "height": h, "points": [], "bounds": []}
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            for j, nu in enumerate([0.0, -0.4, lo0]):
                img = con.accumulate_image(b, nu)
                out[f"{name}/point{j}"] = img.counts.astype(np.uint32)
                rec["points"].append({"nu": bits(nu), "in_image": img.in_image_events,
                                      "contrast": bits(con.image_contrast(img))})
            for j, (lo, hi) in enumerate(ivs):
                ub = con.upper_bound_image(b, VelocityInterval(lo, hi))
                bt = con.bound_terms(b, VelocityInterval(lo, hi))
                out[f"{name}/bound{j}"] = ub.counts.astype(np.uint32)
                rec["bounds"].append({"lo": bits(lo), "hi": bits(hi), "marks": ub.in_image_events,
                                      "c_bar": bits(bt.c_bar)})
            r = sol.maximise_contrast_bnb(b, sol.SolverParams())
            rec["result"] = res_dict(r)
        meta.append(rec)
    np.savez_compressed(os.path.join(HERE, "nonfinite.npz"), **out)
    with open(os.path.join(HERE, "nonfinite.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("nonfinite:", len(meta), "cases")


if __name__ == "__main__":
    big = "--big" in sys.argv
    what = [a for a in sys.argv[1:] if not a.startswith("--")] or ["segments", "images", "bnb", "synth", "evd1", "preproc"]
    if "segments" in what:
        make_segments()
    if "images" in what:
        make_images()
    if "synth" in what:
        make_synth()
    if "evd1" in what:
        make_evd1()
    if "preproc" in what:
        make_preproc()
    if "bnb" in what:
        make_bnb(big)
    if "nonfinite" in what:
        make_nonfinite()
    if "frontier" in what:
        make_frontier()
