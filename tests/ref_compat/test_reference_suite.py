"""The reference's own numerical-path test files, run against the drop-in on the GPU.

SURVEY.md §8(b) "Callers": the drop-in must pass the reference's tests/test_solver.py (and the
other numerical-path files) with the import swapped.  tools/install_reference.sh puts the
unmodified reference package and a copy of its test suite under baseline/_ref (git-ignored; it
travels to the GPU box with the snapshot).  Here pytest runs those files in a subprocess with
tests/ref_compat/dropin_plugin.py, which routes bsesolve's solve-path names to
paper_2601_10557_b200 (dense oracles stay the reference's).  Every test must pass except the
documented deviations below.
"""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[2]
REF_TESTS = ROOT / "baseline" / "_ref" / "ref_tests"

FILES = ["test_solver.py", "test_rayleigh_ritz.py", "test_chebyshev.py", "test_ortho.py", "test_lanczos.py",
         "test_hamiltonian.py"]

# Documented deviations:
DEVIATIONS = {
    # the reference fails this one itself: a 1-ulp tie between |T_12(0)| and |T_12(1)|
    "test_chebyshev.py::TestScalarMatrixConsistency::test_center_gain_is_deeply_damped",
    # north star: shifted CholeskyQR replaces the Householder fallback, method "shifted_cholqr"
    "test_ortho.py::TestCholQr::test_ill_conditioned_falls_back_to_householder",
}


def test_reference_numerical_suite_against_dropin(tmp_path):
    if not REF_TESTS.exists():
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "ref_compat"), str(ROOT / "baseline" / "_ref"),
                                         str(REF_TESTS), str(ROOT), env.get("PYTHONPATH", "")])
    log = tmp_path / "ref_suite.log"
    cmd = [sys.executable, "-m", "pytest", "-q", "-rfE", "-p", "dropin_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(REF_TESTS), *[str(REF_TESTS / f) for f in FILES]]
    out = subprocess.run(cmd, cwd=str(REF_TESTS), env=env, capture_output=True, text=True, timeout=1800)
    text = out.stdout + out.stderr
    log.write_text(text)
    dst = ROOT / "gpurun_out"
    if dst.exists():
        (dst / "ref_suite.log").write_text(text)
    failed = set(re.findall(r"^(?:FAILED|ERROR) (\S+?)(?: - .*)?$", text, re.M))
    failed = {f.split("ref_tests/")[-1] for f in failed}
    unexpected = {f for f in failed if not any(f.startswith(d) for d in DEVIATIONS)}
    summary = text.strip().splitlines()[-1] if text.strip() else ""
    assert re.search(r"\d+ passed", summary), text[-3000:]
    assert not unexpected, f"{summary}\n" + "\n".join(sorted(unexpected)) + "\n" + text[-6000:]
