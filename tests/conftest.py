import json
import os
import sys

import pytest

# several streams per test process (peer-memory SRAD ranks as threads): give
# them their own hardware queues (must be set before CUDA initialises)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run with -m gpu on a B200)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


CORPUS = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested", "bitonic"]


@pytest.fixture(scope="session")
def restatement():
    from oracle import Restatement

    return Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref/libdarm_ref.so not built (make -C oracle ref)")
    return Reference()
