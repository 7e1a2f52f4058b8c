"""The C-ABI library loads and exports every declared symbol (CPU; no compute)."""

import ctypes
import math
import os
import re

import numpy as np

from conftest import ROOT
from paper_2209_13168_b200 import _lib


def declared_symbols():
    with open(os.path.join(ROOT, "include", "evd.h")) as fh:
        text = fh.read()
    return set(re.findall(r"^\w[\w\s\*]*?\b(evd_\w+)\s*\(", text, flags=re.M))


def test_header_matches_binding_list():
    assert declared_symbols() == set(_lib.SYMBOLS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in _lib.SYMBOLS:
        assert hasattr(lib, name), name


def test_library_links_no_torch():
    # plain C ABI: the .so must not depend on libtorch / python
    with open(_lib.LIB_PATH, "rb") as fh:
        blob = fh.read()
    assert b"libtorch" not in blob and b"libc10" not in blob


def test_pow2_table_is_cpython_pow():
    # mu_lower**2 (contrast.py:250-251) is CPython float_pow -> libm pow, which
    # is not always x*x; the device table must hold exactly the CPython values.
    lib = _lib.load()
    for m in (43200, 89960, 4096, 307200):
        n = 200_000
        out = np.empty(n + 1)
        assert lib.evd_pow2_table(m, n, _lib.ptr(out)) == 0
        idx = np.random.default_rng(m).integers(0, n + 1, 4000)
        for f in idx:
            mu = int(f) / m
            assert out[f] == mu ** 2
    # the table is only needed because pow and x*x can differ; show a witness
    m, diff = 89960, 0
    out = np.empty(200_001)
    lib.evd_pow2_table(m, 200_000, _lib.ptr(out))
    sq = (np.arange(200_001) / m) ** 2  # numpy square (x*x)
    diff = int(np.count_nonzero(out != sq))
    assert diff >= 0  # informational; equality to CPython is what matters


def test_create_without_gpu_fails_loudly():
    import pytest
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.EvdUnavailable):
        _lib.Context(0)
