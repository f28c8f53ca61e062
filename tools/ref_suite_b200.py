"""pytest plugin: run the REFERENCE's own test suite with the B200 kernels registered as its backend.

This is the one-branch registration INTEGRATION.md section 1 describes (mx4train/_backend/__init__.py
selecting `paper_2505_14669_b200.kernels`), applied from outside so the installed reference stays
unmodified: every mx4train module that binds `kernels` at import time (codec.py:22, diagnostics.py:19,
hadamard.py:21, qlinear.py:28, quantizers.py:23) gets the B200 module, and `available_backends()` gains
a "b200" entry.

    tools/gpu/ref_suite.sh     (GPU box: baseline/_ref = the pip-installed reference,
                                baseline/_ref_tests = a copy of its pkg/tests, both git-ignored)
"""

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (os.path.join(ROOT, "baseline", "_ref"), ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2505_14669_b200 import kernels as _b200  # noqa: E402

_backend = importlib.import_module("mx4train._backend")
_native = _backend.available_backends().get("native")
_backend.kernels = _b200
_backend.BACKEND = _b200.NAME
_orig_available = _backend.available_backends


def _available():
    out = _orig_available()
    out["b200"] = _b200
    return out


_backend.available_backends = _available
for name in ("codec", "diagnostics", "hadamard", "qlinear", "quantizers"):
    mod = importlib.import_module(f"mx4train.{name}")
    if hasattr(mod, "kernels"):
        mod.kernels = _b200
import mx4train  # noqa: E402

mx4train.BACKEND = _b200.NAME


def pytest_report_header(config):
    return f"mx4train kernels backend: {_backend.kernels.NAME} (paper_2505_14669_b200 on the GPU)"
