"""The per-call entry points keep the window resident (contrast.load_window):
no re-upload for the same arrays, an exact re-upload after any change."""

import numpy as np
import pytest

from oracle import oracle as orc
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import _lib, contrast as con, synth
from paper_2209_13168_b200.geometry import VelocityInterval

pytestmark = pytest.mark.gpu


def test_repeated_calls_do_not_reupload():
    b = synth.random_window(np.random.default_rng(1), 64, 48, 3000)
    ctx = _lib.context()
    evd.bound_terms(b, VelocityInterval(-0.5, -0.3))
    g0 = ctx.window_generation
    for lo, hi in ((-0.5, -0.3), (-1.0, -0.2), (-0.45, -0.44)):
        got = evd.bound_terms(b, VelocityInterval(lo, hi))
        s, mu, cb, fi, _ = orc.bound_terms(b, lo, hi)
        assert (got.s_bar, got.mu_lower, got.c_bar) == (s, mu, cb)
    assert evd.contrast_at(b, -0.4) == orc.contrast_at(b, -0.4)
    assert ctx.window_generation == g0          # nothing uploaded again


def test_in_place_change_is_seen():
    b = synth.random_window(np.random.default_rng(2), 64, 48, 3000)
    ctx = _lib.context()
    iv = VelocityInterval(-0.6, -0.3)
    first = evd.bound_terms(b, iv)
    g0 = ctx.window_generation
    b.x[1234] += 0.75  # same arrays, new contents
    got = evd.bound_terms(b, iv)
    assert ctx.window_generation != g0
    s, mu, cb, fi, _ = orc.bound_terms(b, -0.6, -0.3)
    assert (got.s_bar, got.c_bar) == (s, cb) and got != first


def test_other_window_and_frozen_arrays():
    r = np.random.default_rng(3)
    a = synth.random_window(r, 64, 48, 2000)
    b = synth.random_window(r, 64, 48, 2000)
    for arr in (b.x, b.y, b.t):
        arr.flags.writeable = False
    ctx = _lib.context()
    for batch in (a, b, a, b, b):
        assert evd.contrast_at(batch, -0.3) == orc.contrast_at(batch, -0.3)
    g = ctx.window_generation
    evd.contrast_at(b, -0.2)                     # read-only arrays: identity suffices
    assert ctx.window_generation == g
    # a window replaced behind the cache (another entry point) is re-uploaded
    con.load_window(a, ctx)
    assert evd.contrast_at(b, -0.3) == orc.contrast_at(b, -0.3)
