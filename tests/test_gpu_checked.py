"""The GPU parity suite again on libevd_checked.so (-DEVD_CHECKED: a device
assert on every mark -- inside the frame, p == y * W + x -- and every queue
slot), plus tools/sanitize_paths.py (every device path once against the
oracle).  This stands in for compute-sanitizer, which is closed on the GPU
pool (profiles/sanitizer_r02.txt)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
LIB = os.path.join(ROOT, "paper_2209_13168_b200", "libevd_checked.so")


def _run(args):
    env = dict(os.environ, EVD_LIB=LIB)
    return subprocess.run([sys.executable] + args, cwd=ROOT, env=env, capture_output=True,
                          text=True, timeout=1800)


@pytest.mark.skipif(not os.path.exists(LIB), reason="libevd_checked.so not built")
def test_parity_suite_on_checked_build():
    out = _run(["-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                "--deselect", "tests/test_gpu_checked.py",
                "--deselect", "tests/test_gpu_reference_suite.py", "tests"])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]


@pytest.mark.skipif(not os.path.exists(LIB), reason="libevd_checked.so not built")
def test_every_path_on_checked_build():
    out = _run([os.path.join(ROOT, "tools", "sanitize_paths.py")])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "MISMATCH" not in out.stdout and out.stdout.count(" ok") >= 15, out.stdout
