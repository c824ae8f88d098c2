export DARM_PEER_TIMEOUT_S=30
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.log | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
