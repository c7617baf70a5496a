"""Shared fixtures, the `gpu` marker and the acceptance-criteria summary.

Mirrors the reference's conftest (pkg/tests/conftest.py:16-34): tests record
headline properties through the ``criterion`` fixture and a terminal-summary
hook prints one [PASS]/[FAIL] line per criterion.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

class _Criteria:
    """Headline properties the tests establish, printed as one [PASS]/[FAIL] line each after the run
    (the reference's acceptance-summary output format)."""

    def __init__(self) -> None:
        self.results: dict[str, tuple[str, bool]] = {}

    def __call__(self, key: str, desc: str, ok: bool) -> bool:
        self.results[key] = (desc, bool(ok))
        return bool(ok)

    def lines(self):
        return [f"[{'PASS' if ok else 'FAIL'}] criterion {k}: {d}" for k, (d, ok) in sorted(self.results.items())]


_CRITERIA = _Criteria()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def criterion():
    """record(key, description, ok) -> ok."""
    return _CRITERIA


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    lines = _CRITERIA.lines()
    if lines:
        terminalreporter.section("acceptance criteria")
        for line in lines:
            terminalreporter.write_line(line)


@pytest.fixture(scope="session")
def lib():
    from paper_2411_17089_b200 import _lib

    return _lib.load()


@pytest.fixture(scope="session")
def dev():
    import torch

    torch.cuda.init()
    return torch.device("cuda:0")


GOLDEN = ROOT / "tests" / "golden"
os.environ.setdefault("KVPR_TEST_ROOT", str(ROOT))
