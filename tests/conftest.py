import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle case")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference oracle (oracle/_ref); built on demand here."""
    from oracle import ref as R
    if not R.available():
        import subprocess
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True,
                           stdout=subprocess.DEVNULL)
    if not R.available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return R
