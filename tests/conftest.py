import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session", autouse=True)
def _build_oracle():
    import oracle
    oracle.build()


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# Parity numbers worth keeping in the log of a -q run (the full-size R-14 metrics):
# tests append lines through the `parity_report` fixture, the terminal summary prints them.
_PARITY_LINES = []


@pytest.fixture
def parity_report():
    def add(line):
        print("\n" + line)
        _PARITY_LINES.append(line)
    return add


def pytest_terminal_summary(terminalreporter):
    if _PARITY_LINES:
        terminalreporter.section("parity report")
        for line in _PARITY_LINES:
            terminalreporter.write_line(line)
