import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """A compact record of the full-batch oracle parity checks that ran (tests/test_full_parity.py),
    so a `-q` log still names the layers and modes checked against the CPU oracle."""
    passed = terminalreporter.stats.get("passed", [])
    rows = {}
    for rep in passed:
        nodeid = getattr(rep, "nodeid", "")
        if "test_full_parity.py::" not in nodeid:
            continue
        test, _, param = nodeid.split("::", 1)[1].partition("[")
        rows.setdefault(test, []).append(param.rstrip("]"))
    if not rows:
        return
    terminalreporter.write_line("full-batch oracle parity (tests/test_full_parity.py), passed:")
    for test, params in sorted(rows.items()):
        params = sorted(p for p in params if p) or ["(1 case)"]
        terminalreporter.write_line(f"  {test}: {len(params)} -- " + ", ".join(params))
