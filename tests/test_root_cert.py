"""The root-bound certificate's per-segment cell bound (evd_device.cuh
root_cells_lb, restated here) never exceeds the number of in-frame pixels the
reference rasterisation marks (contrast.py:94-182, via the pinned oracle)."""
import math

import numpy as np

from oracle import oracle as orc


def cells_lb(ax, ay, bx, by, W, H):
    dx, dy = bx - ax, by - ay
    t0, t1 = 0.0, 1.0
    if dx == 0.0:
        if ax < 0.0 or ax > W:
            return 0
    else:
        ta, tb = -ax / dx, (W - ax) / dx
        ta, tb = min(ta, tb), max(ta, tb)
        t0, t1 = max(t0, ta), min(t1, tb)
    if dy == 0.0:
        if ay < 0.0 or ay > H:
            return 0
    else:
        ta, tb = -ay / dy, (H - ay) / dy
        ta, tb = min(ta, tb), max(ta, tb)
        t0, t1 = max(t0, ta), min(t1, tb)
    if not t0 < t1:
        return 0
    x0, x1, y0, y1 = ax + t0 * dx, ax + t1 * dx, ay + t0 * dy, ay + t1 * dy
    m = 1e-6
    xl, xh = max(min(x0, x1), 0.0) + m, min(max(x0, x1), float(W)) - m
    yl, yh = max(min(y0, y1), 0.0) + m, min(max(y0, y1), float(H)) - m
    nx = math.floor(xh) - math.ceil(xl) + 1 if xh > xl else 0
    ny = math.floor(yh) - math.ceil(yl) + 1 if yh > yl else 0
    k = max(nx, ny)
    return k + 1 if k > 0 else 0


def test_cells_lower_bound_vs_reference_rasterisation():
    rng = np.random.default_rng(7)
    W, H = 23, 17
    segs = []
    for _ in range(1500):  # generic, partly outside the frame
        segs.append(tuple(rng.uniform(-10, 35, 4)))
    for _ in range(600):  # integer and half-integer endpoints, axis-parallel, corners
        a = rng.integers(-3, 27, 4) / rng.choice([1, 2], 4)
        if rng.random() < 0.3:
            a[2] = a[0]
        if rng.random() < 0.3:
            a[3] = a[1]
        segs.append(tuple(float(v) for v in a))
    for _ in range(400):  # radial rays through the frame centre (the solve's segments)
        e = rng.integers(0, [W, H])
        s0, s1 = sorted(rng.uniform(0.0, 4.0, 2))
        cx, cy = W / 2.0, H / 2.0
        segs.append((cx + (e[0] - cx) * s0, cy + (e[1] - cy) * s0,
                     cx + (e[0] - cx) * s1, cy + (e[1] - cy) * s1))
    tight = 0
    for ax, ay, bx, by in segs:
        marked = orc.rasterize_segment((ax, ay), (bx, by), W, H)
        inframe = sum(1 for x, y in marked if 0 <= x < W and 0 <= y < H)
        lb = cells_lb(ax, ay, bx, by, W, H)
        assert lb <= inframe, (ax, ay, bx, by, lb, inframe)
        tight += lb > 0
    assert tight > 1000  # the bound is informative, not vacuous
