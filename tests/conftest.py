import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds the oracle (and the executor library if missing) once per session."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)
    lib = os.path.join(REPO, "paper_2005_06787_b200", "libstn_exec.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j8", "-C",
                        os.path.join(REPO, "paper_2005_06787_b200", "csrc")], check=True)
