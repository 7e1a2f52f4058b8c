"""BnB frontiers evaluated as one batch (SURVEY §8(a) part 4, config 3).

``uniform_frontier(domain, depth)`` returns the 2**depth leaves of repeated
``VelocityInterval.split`` (geometry.py:44-46) -- the same floating-point
endpoints the reference's bisection produces (closed forms such as
lo + k*w differ from them).  ``frontier_bounds`` evaluates the
bound of every leaf in one device pass and assembles c_bar exactly as
``contrast.py:248-251``.
"""

from __future__ import annotations

import numpy as np

from .contrast import assemble_bound, frontier_terms
from .events import EventBatch
from .geometry import VelocityInterval


def uniform_frontier(domain: VelocityInterval, depth: int) -> tuple[np.ndarray, np.ndarray]:
    """Leaves of a depth-`depth` bisection of `domain`, left to right."""
    level = [(domain.lo, domain.hi)]
    for _ in range(depth):
        nxt = []
        for lo, hi in level:
            c = 0.5 * (lo + hi)  # VelocityInterval.center
            nxt.append((lo, c))
            nxt.append((c, hi))
        level = nxt
    arr = np.array(level, dtype=np.float64)
    return arr[:, 0].copy(), arr[:, 1].copy()


def frontier_bounds(batch: EventBatch, lo, hi) -> np.ndarray:
    """c_bar of every interval [lo_j, hi_j] (bound_terms(...).c_bar), one pass."""
    s_bar, fi, _ = frontier_terms(batch, lo, hi)
    m = batch.geometry.n_pixels
    return np.array([assemble_bound(int(s), int(f), m).c_bar for s, f in zip(s_bar, fi)])
