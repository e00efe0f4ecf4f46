import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


@pytest.fixture(scope="session")
def built():
    """Native libraries are built in-tree by `make` / __graft_entry__.build()."""
    import subprocess

    subprocess.run(["make", "-s", "-C", ROOT, "tracegen/libtracegen_host.so", "oracle/liboracle.so"], check=True)
    return True
