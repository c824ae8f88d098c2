"""The reference's acceptance criterion 1 (acceptance.cpp:101-119) through the
reference-side C++ binding include/darm_gpu.hpp: for every positive corpus
kernel, warp sizes {4, 8, 32, 64} and 100 makeRandomInput fixtures, the
reference's compareRuns finds the sm_100a unmelded and melded results equal
to the reference interpreter's (oracle/bridge_test.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

BRIDGE = os.path.join(ROOT, "oracle", "_ref", "bridge_test")


@pytest.mark.gpu
def test_acceptance_c1_on_gpu_through_reference_types():
    if not os.path.exists(BRIDGE):
        pytest.skip("oracle/_ref/bridge_test not built (make -C oracle ref bridge, needs /root/reference)")
    r = subprocess.run([BRIDGE, "100"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "compareRuns verdicts equal" in r.stdout
