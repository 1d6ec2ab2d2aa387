"""pytest plugin: apply the B200 drop-in to the UNMODIFIED reference before its
own test modules are collected (they bind ``from signadd import ndft, ...`` at
import time).  Loaded by tests/test_ref_conformance.py as
``-p dropin_plugin`` on the reference's suite in baseline/_ref/ref_tests.

SA_DROPIN_MF=1 also patches ``mf_complex`` (for test_operator.py); by default it
stays on the CPU because the reference's test oracles (tests/oracles.py:10)
call it to check the transforms.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (os.path.join(ROOT, "baseline", "_ref"), ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import signadd  # noqa: E402  (the reference, from baseline/_ref)

from paper_1402_0532_b200 import dropin  # noqa: E402

if not signadd.__file__.startswith(os.path.join(ROOT, "baseline", "_ref")):
    raise RuntimeError(f"reference imported from {signadd.__file__}, not baseline/_ref")
dropin.install(signadd, mf_complex=os.environ.get("SA_DROPIN_MF") == "1")
assert signadd.ndft.__module__ == "paper_1402_0532_b200.dropin"


def pytest_report_header(config):
    mf = " + mf_complex" if os.environ.get("SA_DROPIN_MF") == "1" else ""
    return f"B200 drop-in installed into {signadd.__file__} (ndft, nfft, ... {mf})"
