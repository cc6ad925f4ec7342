"""The drop-in check: the REFERENCE package's own test suite
(/root/reference/pkg/tests, run in place, read-only) against this backend's
mirror of its API, with ``import lego`` redirected by tests/lego_shim_plugin.py.

Excluded: ``test_cli.py`` (the CLI is out of scope).
Expected failure: one test that asserts a *weakness* of the reference
simplifier (plain ``simplify`` cannot recompose ``2*(4*(x//8) + t) + x%8``
without expansion; this backend's normal-form engine can).
Skipped where the reference is absent (the GPU box)."""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
EXPECTED_FAIL = {"test_simplify.py::test_best_variant_prefers_expansion_when_it_unlocks_recompose"}


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference package not present")
def test_reference_suite_against_the_mirror(tmp_path):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", PYTHONPATH=HERE)
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "lego_shim_plugin", "-p", "no:cacheprovider",
                        "-q", "-rf", REF_TESTS, f"--ignore={REF_TESTS}/test_cli.py"],
                       capture_output=True, text=True, timeout=600, cwd=tmp_path, env=env)
    failed = {ln.split(" ")[1].split("tests/")[-1] for ln in r.stdout.splitlines() if ln.startswith("FAILED ")}
    summary = [ln for ln in r.stdout.splitlines() if " passed" in ln or " failed" in ln]
    assert failed == EXPECTED_FAIL, (failed, summary, r.stdout[-3000:])
    passed = int(summary[-1].split(" passed")[0].split()[-1])
    assert passed >= 212, summary
