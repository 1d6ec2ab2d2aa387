"""The reference's OWN test suite, unmodified, run with the B200 drop-in applied
(VERDICT r1 "do this" 1).

tools/install_ref.sh (called by __graft_entry__.build()) pip-installs the
unmodified reference into baseline/_ref and copies its tests/ next to it
(baseline/_ref/ref_tests, git-ignored, travels to the GPU box).  Each module
runs in a subprocess so that tests/dropin_plugin.py can patch ``signadd``
before collection.  test_operator.py runs with ``mf_complex`` patched as well;
the other modules keep it on the CPU, where the reference's oracles
(tests/oracles.py) use it as the checker.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="baseline/_ref/ref_tests absent (run tools/install_ref.sh)")

# module -> (patch mf_complex too, expected outcome counts from the reference's own CPU run)
MODULES = {
    "test_operator.py": True,
    "test_transforms.py": False,
    "test_ambiguity.py": False,
    "test_detection.py": False,
    "test_acceptance.py": False,
    "test_cli.py": False,
}


def run_ref_module(mod: str, mf: bool, timeout=900):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), REF, ROOT, env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["SA_DROPIN_MF"] = "1" if mf else "0"
    cmd = [sys.executable, "-m", "pytest", os.path.join(REF_TESTS, mod), "-q", "-p", "dropin_plugin",
           "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-o", "addopts=", "-rfEx"]
    p = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


def counts(text):
    out = {}
    for n, what in re.findall(r"(\d+) (passed|failed|xfailed|skipped|errors?|xpassed)", text):
        out[what] = int(n)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("mod", list(MODULES))
def test_reference_suite_through_dropin(mod, sa):
    rc, text = run_ref_module(mod, MODULES[mod])
    c = counts(text.splitlines()[-1] if text.strip() else "")
    print(f"{mod}: {c}")
    assert "B200 drop-in installed" in text, text[-3000:]
    assert rc == 0 and c.get("failed", 0) == 0 and not c.get("error") and not c.get("errors"), text[-6000:]
    assert c.get("passed", 0) > 0


def test_plugin_patches_reference_cpu():
    """CPU: the plugin imports the reference from baseline/_ref and installs the
    drop-in bindings (no compute call)."""
    code = ("import dropin_plugin, signadd, signadd.cli as c; "
            "assert signadd.ndft.__module__ == 'paper_1402_0532_b200.dropin'; "
            "assert c._TRANSFORMS['nfft'] is signadd.nfft; print('ok')")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), REF, ROOT, env.get("PYTHONPATH", "")])
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ok" in p.stdout, p.stderr[-2000:]
