"""The reference's OWN test suite, unmodified, run with the B200 drop-in applied
(VERDICT r1 "do this" 1).

tools/install_ref.sh (called by __graft_entry__.build()) pip-installs the
unmodified reference into baseline/_ref and copies its tests/ next to it
(baseline/_ref/ref_tests, git-ignored, travels to the GPU box) together with
the reference's own recorded CPU run (pkg/test_output.txt).  Each module runs
in a subprocess so that tests/dropin_plugin.py patches ``signadd`` before
collection.  test_operator.py runs with ``mf_complex`` patched as well; the
other modules keep it on the CPU, where the reference's oracles
(tests/oracles.py) use it as the checker.

Pass criterion: every test's outcome equals the reference's own recorded
outcome (PASSED / XFAIL / FAILED), and the assertion messages of the tests the
reference itself fails (test_acceptance.py criteria 6 and 7: detection counts
and side-lobe floors over 10 seeds) are identical -- the drop-in reproduces
the reference's detections and floors exactly, failures included.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")
RECORDED = os.path.join(REF_TESTS, "reference_test_output.txt")

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="baseline/_ref/ref_tests absent (run tools/install_ref.sh)")

# module -> also patch mf_complex
MODULES = {
    "test_operator.py": True,
    "test_transforms.py": False,
    "test_ambiguity.py": False,
    "test_detection.py": False,
    "test_acceptance.py": False,
    "test_cli.py": False,
}

_OUTCOME = re.compile(r"^(?:tests/)?(test_\w+\.py)::(\S+) (PASSED|FAILED|XFAIL|XPASS|SKIPPED|ERROR)\b")
_ASSERT = re.compile(r"^E\s+(AssertionError: .*)$")


def _env(mf: bool):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), REF, ROOT, env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["SA_DROPIN_MF"] = "1" if mf else "0"
    return env


def run_ref_module(mod: str, mf: bool, timeout=900):
    cmd = [sys.executable, "-m", "pytest", os.path.join(REF_TESTS, mod), "-v", "-p", "dropin_plugin",
           "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-o", "addopts=", "--tb=short"]
    p = subprocess.run(cmd, cwd=REF_TESTS, env=_env(mf), capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


def parse(text, mod):
    outcomes, asserts = {}, []
    for line in text.splitlines():
        m = _OUTCOME.match(line.strip())
        if m and m.group(1) == mod:
            outcomes[m.group(2)] = m.group(3)
        a = _ASSERT.match(line.rstrip())
        if a:
            asserts.append(a.group(1).strip())
    return outcomes, asserts


def recorded(mod):
    """The reference's own CPU outcomes for ``mod`` and its assertion messages."""
    text = open(RECORDED).read()
    out, _ = parse(text, mod)
    # assertion messages belong to the failure sections of this module
    asserts = []
    sections = re.split(r"^_{5,} ", text, flags=re.M)
    for sec in sections[1:]:
        name = sec.split(" ", 1)[0]
        if name in out and out[name] == "FAILED":
            asserts += [a.group(1).strip() for a in map(_ASSERT.match, sec.splitlines()) if a]
    return out, asserts


@pytest.mark.gpu
@pytest.mark.parametrize("mod", list(MODULES))
def test_reference_suite_through_dropin(mod, sa):
    rc, text = run_ref_module(mod, MODULES[mod])
    assert "B200 drop-in installed" in text, text[-3000:]
    got, got_asserts = parse(text, mod)
    want, want_asserts = recorded(mod)
    summary = {k: sum(1 for v in got.values() if v == k) for k in sorted(set(got.values()))}
    print(f"{mod}: {summary} (reference recorded {len(want)} tests)")
    assert got, text[-3000:]
    assert set(got) == set(want), (sorted(set(got) ^ set(want)), text[-3000:])
    diff = {k: (got[k], want[k]) for k in got if got[k] != want[k]}
    assert not diff, (diff, text[-6000:])
    assert sorted(got_asserts) == sorted(want_asserts), (got_asserts, want_asserts)
    assert (rc == 0) == all(v != "FAILED" for v in want.values())


def test_recorded_outcomes_parse():
    """CPU: the reference's recorded run parses into the expected totals (the
    suite's 212 tests; criteria 6 and 7 of test_acceptance.py fail there)."""
    if not os.path.exists(RECORDED):
        pytest.skip("recorded reference run absent")
    tot = {}
    for mod in MODULES:
        out, asserts = recorded(mod)
        tot[mod] = out
        if mod == "test_acceptance.py":
            assert {k for k, v in out.items() if v == "FAILED"} == {
                "test_criterion_6_contaminated_robustness_trend", "test_criterion_7_awgn_trend"}
            assert len(asserts) == 2 and "eq12a detected 0/10" in asserts[0]
    assert sum(len(v) for v in tot.values()) > 150


def test_plugin_patches_reference_cpu():
    """CPU: the plugin imports the reference from baseline/_ref and installs the
    drop-in bindings (no compute call)."""
    code = ("import dropin_plugin, signadd, signadd.cli as c; "
            "assert signadd.ndft.__module__ == 'paper_1402_0532_b200.dropin'; "
            "assert c._TRANSFORMS['nfft'] is signadd.nfft; print('ok')")
    p = subprocess.run([sys.executable, "-c", code], env=_env(False), capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ok" in p.stdout, p.stderr[-2000:]
