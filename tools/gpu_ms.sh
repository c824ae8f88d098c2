set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "merge or abi" > gpurun_out/pytest_ms.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ms.log
timeout 300 python tools/time_ms.py 1048576 16777216 > gpurun_out/time_ms.log 2>&1
