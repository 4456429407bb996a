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


# A kernel that never finishes would block pytest inside a CUDA call, where pytest-timeout's
# signal cannot interrupt it.  For GPU tests a watchdog thread ends the process instead, so a
# hang shows up as a failed run rather than a stalled one.
_WATCHDOG_S = float(os.environ.get("BSORT_TEST_WATCHDOG_S", "900"))


@pytest.fixture(autouse=True)
def _gpu_watchdog(request):
    if request.node.get_closest_marker("gpu") is None:
        yield
        return
    import threading
    done = threading.Event()

    def watch():
        if not done.wait(_WATCHDOG_S):
            sys.stderr.write(f"\nwatchdog: {request.node.nodeid} exceeded {_WATCHDOG_S}s, aborting\n")
            sys.stderr.flush()
            os._exit(3)

    t = threading.Thread(target=watch, daemon=True)
    t.start()
    try:
        yield
    finally:
        done.set()
