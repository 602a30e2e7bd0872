"""The reference's OWN test files run against the reference package with its averaging
path routed through libringmix_b200 by the INTEGRATION binding (integration/ringmix_b200.py:
permutation_for_step, apply_mixing and the fused _gossip_step on the reference's (d, L)
float64 arrays).  The unmodified reference is installed under baseline/_ref by
tools/install_reference.sh together with a copy of its tests (pkg/tests); the run is
skipped where that install is absent."""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"
TESTS = REF / "ringmix_ref_tests"
FAST = ["test_seeding.py", "test_mixing.py", "test_simulation.py", "test_spectral.py",
        "test_objectives.py", "test_harness.py"]


def _run(files, timeout):
    if not (REF / "ringmix").is_dir() or not TESTS.is_dir():
        pytest.skip("reference not installed under baseline/_ref (tools/install_reference.sh)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF), str(ROOT / "integration")]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "pytest_ringmix_b200", "-p",
           "no:cacheprovider", "--rootdir", str(TESTS)] + [str(TESTS / f) for f in files]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env,
                       cwd=str(TESTS))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    m = re.search(r"RINGMIX_B200_CALLS (.*)", out)
    assert m, out[-2000:]
    calls = dict(kv.split("=") for kv in m.group(1).split())
    return out, {k: int(v) for k, v in calls.items()}


def test_reference_unit_tests_through_the_binding():
    out, calls = _run(FAST, 900)
    # the averaging path really went through the GPU
    assert calls["permutation_for_step"] > 0 and calls["apply_mixing"] > 0
    assert calls["gossip_step"] > 0
    summary = [x for x in out.splitlines() if re.search(r"\d+ passed", x)]
    print(summary[-1] if summary else out[-500:], calls)


@pytest.mark.slow
def test_reference_acceptance_criteria_through_the_binding():
    out, calls = _run(["test_acceptance.py"], 1800)
    assert calls["gossip_step"] > 0
    crit = re.findall(r"\[criterion (\d+)\] .*: (PASS|FAIL)", out)
    assert crit and all(v == "PASS" for _, v in crit), crit
