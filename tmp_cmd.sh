export DARM_PEER_TIMEOUT_S=20
timeout 900 python -m pytest tests/test_srad_peer.py -q -m gpu -k thin > gpurun_out/pytest_peer.log 2>&1; echo "peer tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/pytest_peer.log | tail -20
