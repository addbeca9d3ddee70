"""The reference package's own hot-path tests, run through the drop-in on the
GPU: polygrain's test_objective.py, test_acceptance.py (criteria 1-10) and
test_optimizer.py
with polygrain.objective / polygrain.optimizer routed to
paper_2605_20816_b200 (tests/refsuite/pgx_dropin.py).

Needs the reference installed once into baseline/_ref (git-ignored, shipped
to the GPU box with the repo snapshot): skipped without it.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "polygrain_tests")


@pytest.mark.parametrize("suite", ["test_objective.py", "test_acceptance.py", "test_optimizer.py"])
def test_reference_suite_through_dropin(suite, tmp_path):
    if not os.path.exists(os.path.join(REF_TESTS, suite)):
        pytest.skip("reference package not installed into baseline/_ref")
    report = tmp_path / "calls.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests", "refsuite")]),
               PGX_DROPIN_REPORT=str(report), PGX_PRECISION="exact")
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "pgx_dropin",
                           "-p", "no:cacheprovider", "--rootdir", REF_TESTS, os.path.join(REF_TESTS, suite)],
                          cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1800)
    tail = (proc.stdout + proc.stderr)[-4000:]
    assert proc.returncode == 0, tail
    calls = json.loads(report.read_text())
    print(suite, proc.stdout.strip().splitlines()[-1], calls)
    assert sum(calls.values()) > 0, calls  # the reference tests really went through the drop-in
    if suite == "test_objective.py":
        for name in ("objective", "gradient", "soft_assign", "evaluate_objective"):
            assert calls[name] > 0, (name, calls)
