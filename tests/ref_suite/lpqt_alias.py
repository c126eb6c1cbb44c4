"""pytest plugin: run the REFERENCE's own test suite against the drop-in.

    python -m pytest -p tests.ref_suite.lpqt_alias baseline/_ref/tests

Loaded before collection, it makes `import lpqt` / `from lpqt.cli import ...`
resolve to `paper_2312_08583_b200` (the B200 package) and its modules, so the
reference tests (pkg/tests/test_*.py, staged next to the installed reference
by tools/install_reference.sh; never committed) exercise the drop-in exactly
as they exercise `lpqt` 0.1.0.  The reference package itself is not
importable in that run (baseline/_ref is not on sys.path).
"""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

MODULES = ("codec", "quantizer", "packing", "dequant", "gemm", "container", "cli", "errors")


def install() -> None:
    pkg = importlib.import_module("paper_2312_08583_b200")
    sys.modules["lpqt"] = pkg
    for m in MODULES:
        sys.modules[f"lpqt.{m}"] = importlib.import_module(f"paper_2312_08583_b200.{m}")


install()


def pytest_configure(config):
    """Create the CUDA context and load the library before any test runs: the
    reference suite holds a few criteria to wall-clock budgets of ~1 s
    (tests/test_acceptance.py `_Budget`), which measure the computation, not
    this process's one-time GPU start-up (the reference, pure numpy, has none)."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        return
    if torch.cuda.is_available():
        pkg = sys.modules["lpqt"]
        pkg.encode_rtn(pkg.FP6_E3M2, 1.0)
        torch.cuda.synchronize()
