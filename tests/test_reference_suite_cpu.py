"""The reference's OWN test suite run unmodified against this package (drop-in proof, CPU).

tests/refshim maps the reference's package name (`kvoverlap.costmodel`, `.hwprofile`, `.scheduler`,
`.pipesim`, `.cli`, `.numerics`) onto this package's modules, plus a `kvoverlap` console script; the
test files are read from /root/reference/pkg/tests (present in the build container only -- skipped
elsewhere; nothing is copied).  Deselected, because this package runs them on the GPU: the
reference's fp64 NumPy numerics tests (test_numerics.py, acceptance criterion 07, `validate`) --
their device counterparts are tests/test_numerics_gpu.py and criterion N1."""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

from .conftest import ROOT

REF_TESTS = Path("/root/reference/pkg/tests")
FILES = ["test_costmodel.py", "test_hwprofile.py", "test_scheduler.py", "test_pipesim.py", "test_cli.py",
         "test_acceptance.py"]
DESELECT = "not criterion_07 and not test_validate_ok and not test_validation_cases_all_pass"


@pytest.mark.skipif(not REF_TESTS.is_dir(), reason="reference test suite not present (GPU box)")
def test_reference_suite_passes_against_this_package(criterion):
    shim = ROOT / "tests" / "refshim"
    env = dict(os.environ, PYTHONPATH=f"{shim}{os.pathsep}{ROOT}", PATH=f"{shim / 'bin'}{os.pathsep}{os.environ['PATH']}")
    probe = subprocess.run([sys.executable, "-c", "import kvoverlap.costmodel as c, kvoverlap.pipesim as p; "
                            "print(c.opt_preset.__module__, p.simulate.__module__)"],
                           capture_output=True, text=True, env=env, cwd=ROOT)
    assert probe.stdout.split() == ["paper_2411_17089_b200.costmodel", "paper_2411_17089_b200.pipesim"], probe
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-k", DESELECT,
                          *[str(REF_TESTS / f) for f in FILES]],
                         capture_output=True, text=True, env=env, cwd=ROOT, timeout=1200)
    tail = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    m = re.search(r"(\d+) passed", tail)
    passed = int(m.group(1)) if m else 0
    ok = out.returncode == 0 and "failed" not in tail and passed >= 145
    assert criterion("R1", f"the reference's own tests ({', '.join(FILES)}) against this package: {tail}", ok), \
        out.stdout[-3000:]


@pytest.mark.skipif(not REF_TESTS.is_dir(), reason="reference test suite not present (GPU box)")
def test_reference_numerics_tests_pin_the_oracle(criterion):
    """The reference's own fp64 numerics tests (test_numerics.py, acceptance criterion 07: split rebuild
    exact within 1e-12 over 1008 randomized checks) run against oracle/numerics_ref.py through
    tests/refshim_oracle -- the oracle every GPU parity test is judged against passes the reference's
    own exactness tests, beside the npz goldens (tests/test_oracle_cpu.py)."""
    shim = ROOT / "tests" / "refshim_oracle"
    env = dict(os.environ, PYTHONPATH=f"{shim}{os.pathsep}{ROOT}")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          str(REF_TESTS / "test_numerics.py"),
                          str(REF_TESTS / "test_acceptance.py") + "::test_criterion_07_split_rebuild_is_exact"],
                         capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    tail = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    m = re.search(r"(\d+) passed", tail)
    ok = out.returncode == 0 and "failed" not in tail and m is not None and int(m.group(1)) >= 15
    assert criterion("R2", f"the reference's numerics tests (test_numerics.py + criterion 07) against the oracle: "
                           f"{tail}", ok), out.stdout[-3000:]
