mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "lud" > gpurun_out/pytest_lud.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lud.log
timeout 300 python tools/time_lud.py 2048 8192 > gpurun_out/time_lud.log 2>&1
