import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE.json sizes)")


def _make(target):
    subprocess.run(["make", "-s", "-C", REPO, target], check=True)


@pytest.fixture(scope="session", autouse=True)
def _built_oracle():
    # The oracle is test infrastructure: build it once per session (cheap, plain C).
    if not os.path.exists(os.path.join(REPO, "oracle", "liboracle.so")):
        _make("oracle")


def parse_golden(name):
    """Parse a tests/golden/*.txt fixture: `key v1 v2 ...` lines, '#' comments."""
    out = {}
    with open(os.path.join(REPO, "tests", "golden", name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            out[key] = vals
    return out
