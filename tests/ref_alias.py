"""pytest plugin: run the reference's OWN test files against the drop-in.

Loaded with ``-p ref_alias`` by tests/test_gpu_reference_suite.py.  The
reference package ``eventdiv`` (baseline/_ref, installed unmodified by
tools/install_reference.sh) is imported with its hot-path modules replaced by
this repo's: ``eventdiv.geometry`` (the warp), ``eventdiv.contrast`` (images
and bounds) and ``eventdiv.solver`` (the BnB) are paper_2209_13168_b200's, so
the reference's own events / simulator / evaluate modules -- and every test --
call the B200 path, exactly as a user switching packages would.  Its plots
module needs matplotlib (absent in the image) and is out of scope: a no-op
stand-in keeps ``eventdiv.cli`` importable.
"""

import importlib.util
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2209_13168_b200 import contrast, geometry, solver  # noqa: E402

spec = importlib.util.find_spec("eventdiv")
assert spec is not None and spec.origin.startswith(REF), spec
pkg = importlib.util.module_from_spec(spec)
sys.modules["eventdiv"] = pkg
for name, mod in (("geometry", geometry), ("contrast", contrast), ("solver", solver)):
    sys.modules["eventdiv." + name] = mod
plots = types.ModuleType("eventdiv.plots")
plots.plot_divergence_timeline = lambda *a, **k: None
plots.plot_evaluation_report = lambda *a, **k: None
sys.modules["eventdiv.plots"] = plots
spec.loader.exec_module(pkg)
for name, mod in (("geometry", geometry), ("contrast", contrast), ("solver", solver),
                  ("plots", plots)):
    setattr(pkg, name, mod)
assert pkg.maximise_contrast_bnb is solver.maximise_contrast_bnb
