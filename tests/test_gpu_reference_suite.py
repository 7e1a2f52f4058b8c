"""The reference's own tests (pkg/tests, copied unmodified into
baseline/_ref/reference_tests by tools/install_reference.sh) run against the
drop-in on the GPU: ``eventdiv.geometry / contrast / solver`` are this repo's
modules (tests/ref_alias.py).  Covers test_geometry.py, test_contrast.py,
test_solver.py and acceptance criteria 1-5 and 7 (test_acceptance.py: bound
validity on 1,000 random cases, BnB vs a 4096-point grid on 50 batches,
divergence recovery, runtime proxy, contrast sanity, 10,000 segments vs the
exhaustive oracle).  Out of scope and deselected: write_pgm (a debug dump) and
the CLI / plotting criteria 6 and 8 (flow-file evaluation, CLI determinism)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
TESTS = os.path.join(ROOT, "baseline", "_ref", "reference_tests")


@pytest.mark.skipif(not os.path.isdir(TESTS), reason="run tools/install_reference.sh")
@pytest.mark.parametrize("target", [
    "test_geometry.py", "test_contrast.py", "test_solver.py",
    "test_acceptance.py::test_criterion_1_bound_validity",
    "test_acceptance.py::test_criterion_2_global_optimality",
    "test_acceptance.py::test_criterion_3_divergence_recovery",
    "test_acceptance.py::test_criterion_4_runtime_proxy",
    "test_acceptance.py::test_criterion_5_contrast_sanity",
    "test_acceptance.py::test_criterion_7_rasterization_oracle"])
def test_reference_suite_through_drop_in(target):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), TESTS, ROOT]),
               NUMBA_CACHE_DIR="/tmp/evd_numba_cache", PYTHONDONTWRITEBYTECODE="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-s", "-p", "ref_alias",
                          "-p", "no:cacheprovider", "--rootdir", TESTS,
                          "--deselect", "test_contrast.py::TestPgm::test_write",
                          os.path.join(TESTS, target)],
                         cwd=TESTS, env=env, capture_output=True, text=True, timeout=1200)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and "failed" not in out.stdout.split("\n")[-2], tail
